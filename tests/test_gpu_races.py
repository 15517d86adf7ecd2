"""Race screening for the shared-memory pipelines (SURVEY §5 "race detection"), without compute-sanitizer.

compute-sanitizer (racecheck / synccheck / memcheck) is closed on the GPU pool: earlier runs under it left
GPUs needing a reset (`tools/sanitize_cases.py` is the case list for a box where it runs). What these tests
do instead: a data race in an mbarrier / cp.async / TMA ring or in a split-K reduction changes WHICH values
meet in a sum, so it shows as a wrong result or as a run-to-run difference. Every pipelined kernel path is
run REPS times on uniform [-1, 1) inputs (sums that are sensitive to the last bit), each time with an
HBM- and SM-heavy kernel running concurrently on another stream to shift the timing, and every repetition
must be bit-identical to the first one and within 1e-12 normwise of the host oracle.
"""
import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

SEED = 1910
REPS = 16
TOL = 1e-12


@pytest.fixture(scope="module")
def dbm():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1910_04796_b200 as d

    d.load()
    return d


@pytest.fixture(scope="module")
def ctx(dbm):
    c = dbm.Context()
    yield c
    c.close()


def host(t):
    return t.detach().to("cpu").numpy().copy()


def perturb(n=1 << 26):
    """Queue HBM / SM work on a side stream (overlaps the multiply that follows on the ctx stream)."""
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        x = torch.rand(n, device="cuda", dtype=torch.float64)
        for _ in range(4):
            x = x * 1.0000001 + 0.5
    return s, x


def repeat(dbm, ctx, make, path):
    outs = []
    for _ in range(REPS):
        A, B, C = make()
        A.fill_random(SEED, 0, 0)
        B.fill_random(SEED, 1, 0)
        C.fill_random(SEED, 2, 0)
        s, x = perturb()
        dbm.multiply(ctx, 0.75, A, B, -1.25, C, path)
        ctx.sync()
        s.synchronize()
        del x
        outs.append(host(C.arena)[: C.arena_bytes // 8])
    for o in outs[1:]:
        assert np.array_equal(o, outs[0])
    return outs[0]


# (label, M, N, K, bs, path): the kernel each one reaches
DENSE = [
    ("dgemm bs 64 (zero-copy B)", 704, 704, 1408, 64, "densified"),
    ("dgemm bs 22", 704, 528, 1100, 22, "densified"),
    ("smm22q 4x4 squares", 704, 704, 704, 22, "blocked"),
    ("smm22 groups / mixed", 198, 110, 264, 22, "blocked"),
    ("smm22q split-K, few long runs", 88, 88, 45056, 22, "blocked"),
    ("smm64 TMA", 512, 512, 640, 64, "blocked"),
    ("run kernel bs 13", 260, 208, 338, 13, "blocked"),
    ("run squares bs 5", 1280, 1280, 40, 5, "blocked"),
]


@pytest.mark.parametrize("label,M,N,K,bs,path", DENSE, ids=[d[0] for d in DENSE])
def test_dense_paths_repeat_bit_identical(dbm, ctx, orc, label, M, N, K, bs, path):
    got = repeat(dbm, ctx, lambda: (dbm.Matrix(ctx, M, K, bs), dbm.Matrix(ctx, K, N, bs), dbm.Matrix(ctx, M, N, bs)),
                 path)
    Ao, Bo = orc.fill_arena(SEED, 0, 0, M, K, bs), orc.fill_arena(SEED, 1, 0, K, N, bs)
    Co = orc.fill_arena(SEED, 2, 0, M, N, bs)
    orc.multiply_blocked(M // bs, N // bs, K // bs, bs, 0.75, Ao, Bo, -1.25, Co)
    assert np.linalg.norm(got - Co) <= TOL * max(np.linalg.norm(Co), 1.0)


@pytest.mark.parametrize("bs,occ", [(22, 0.3), (64, 0.4), (5, 0.5)])
def test_sparse_paths_repeat_bit_identical(dbm, ctx, bs, occ):
    n = 32 * bs
    Mb = n // bs

    def make():
        return (dbm.Matrix(ctx, n, n, bs, mask=dbm.pattern_random(3, 0, Mb, Mb, occ)),
                dbm.Matrix(ctx, n, n, bs, mask=dbm.pattern_random(3, 1, Mb, Mb, occ)),
                dbm.Matrix(ctx, n, n, bs, mask=dbm.pattern_random(3, 2, Mb, Mb, 0.8)))

    repeat(dbm, ctx, make, "blocked")


@pytest.mark.parametrize("path", ["blocked", "densified"])
def test_nonuniform_paths_repeat_bit_identical(dbm, ctx, path):
    cyc = [5, 13, 23, 26, 32]
    rs = [cyc[i % 5] for i in range(40)]
    ks = [cyc[(i + 2) % 5] for i in range(37)]
    cs = [cyc[(i + 4) % 5] for i in range(35)]

    def make():
        return (dbm.Matrix(ctx, 0, 0, 0, row_sizes=rs, col_sizes=ks),
                dbm.Matrix(ctx, 0, 0, 0, row_sizes=ks, col_sizes=cs),
                dbm.Matrix(ctx, 0, 0, 0, row_sizes=rs, col_sizes=cs))

    repeat(dbm, ctx, make, path)


def test_sanitize_case_list_exists():
    """The compute-sanitizer case list stays runnable for a box where the sanitizer is allowed."""
    assert os.path.exists(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools",
                                       "sanitize_cases.py"))
