"""GPU parity for non-uniform block sizes (reading R16) through the C ABI, against the
host oracle (orc_nu_*, pinned in test_oracle_pins.py): fill, block access, densify / undensify bit-exact;
multiplies of mixed (m, n, k) block products on both local paths <= 1e-12 normwise, bit-exact with integer
inputs; block-sparse non-uniform operands on the densified path; stack lists; partition validation."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

SEED = 1910
TOL = 1e-12

# block-size mixes: CP2K-like basis-set sizes (5, 13, 23, 26 ...), the paper's 22 / 64, ragged tails
MIXES = {
    "cp2k": ([5, 13, 23, 26, 13, 5, 32, 9], [13, 26, 5, 23, 9, 32], [23, 5, 26, 13, 32, 9, 5]),
    "paper": ([22, 64, 22, 64, 22], [64, 22, 64], [22, 22, 64, 64, 22, 64]),
    "tiny": ([1, 2, 3], [4, 1], [2, 7, 1, 3]),
    "wide_k": ([8, 16], [24, 8, 16], [3, 61, 40, 2, 17]),
}


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
    torch.cuda.synchronize()
    return t.detach().cpu().numpy()


def nu(dbm, ctx, rs, cs, mask=None):
    return dbm.Matrix(ctx, 0, 0, 0, row_sizes=rs, col_sizes=cs, mask=mask)


@pytest.mark.parametrize("mix", sorted(MIXES))
def test_nu_fill_and_blocks_bit_exact(dbm, ctx, orc, mix):
    ms, ns, _ = MIXES[mix]
    m = nu(dbm, ctx, ms, ns)
    m.fill_random(SEED, 2, 0)
    D = orc.fill_dense(SEED, 2, 0, sum(ms), sum(ns))
    assert np.array_equal(host(m.arena)[: m.arena_bytes // 8], orc.nu_scatter(D, ms, ns))
    ro, co = np.concatenate([[0], np.cumsum(ms)]), np.concatenate([[0], np.cumsum(ns)])
    for bi, bj in [(0, 0), (len(ms) - 1, len(ns) - 1), (1, len(ns) // 2)]:
        blk = m.get_block(bi, bj)
        assert blk.shape == (ms[bi], ns[bj])
        assert np.array_equal(blk, D[ro[bi]:ro[bi + 1], co[bj]:co[bj + 1]])
    new = np.arange(ms[1] * ns[0], dtype=np.float64).reshape(ms[1], ns[0])
    m.set_block(1, 0, new)
    assert np.array_equal(m.get_block(1, 0), new)


@pytest.mark.parametrize("layout", [0, 1])
@pytest.mark.parametrize("sparse", [False, True])
def test_nu_densify_undensify_bit_exact(dbm, ctx, orc, layout, sparse):
    ms, ns, _ = MIXES["cp2k"]
    mask = orc.pattern_random(3, 0, len(ms), len(ns), 0.6) if sparse else None
    m = nu(dbm, ctx, ms, ns, mask)
    m.fill_random(SEED, 0, 0)
    M, N = sum(ms), sum(ns)
    D = orc.fill_dense(SEED, 0, 0, M, N)
    if sparse:  # absent blocks densify to zeros
        keep = np.zeros((M, N), bool)
        ro, co = np.concatenate([[0], np.cumsum(ms)]), np.concatenate([[0], np.cumsum(ns)])
        for bi in range(len(ms)):
            for bj in range(len(ns)):
                keep[ro[bi]:ro[bi + 1], co[bj]:co[bj + 1]] = mask[bi, bj]
        D = np.where(keep, D, 0.0)
    ld = (M if layout == 0 else N) + 3
    dense = torch.full((ld * (N if layout == 0 else M),), float("nan"), dtype=torch.float64, device="cuda")
    m.densify(dense, ld, layout)
    got = host(dense).reshape(-1, ld)
    got = got[:, :M].T if layout == 0 else got[:, :N]
    assert np.array_equal(got, D)
    # undensify with alpha / beta: two roundings per element, stored blocks only
    Dn = np.random.default_rng(1).uniform(-1, 1, (M, N))
    before = orc.nu_scatter(D, ms, ns, mask=mask)
    m.undensify(torch.from_numpy(np.ascontiguousarray(Dn.T)).reshape(-1).cuda(), 0.75, -1.25, M)
    exp = 0.75 * orc.nu_scatter(Dn, ms, ns, mask=mask) + (-1.25) * before
    assert np.array_equal(host(m.arena)[: m.arena_bytes // 8], exp)


def run_nu(dbm, ctx, orc, mix, path, alpha, beta, kind=0, masks=(None, None, None)):
    ms, ns, ks = MIXES[mix] if isinstance(mix, str) else mix
    A, B, C = nu(dbm, ctx, ms, ks, masks[0]), nu(dbm, ctx, ks, ns, masks[1]), nu(dbm, ctx, ms, ns, masks[2])
    A.fill_random(SEED, 0, kind)
    B.fill_random(SEED, 1, kind)
    C.fill_random(SEED, 2, kind)
    st = dbm.multiply(ctx, alpha, A, B, beta, C, path)
    got = host(C.arena)[: C.arena_bytes // 8]
    Ad = orc.fill_dense(SEED, 0, kind, sum(ms), sum(ks))
    Bd = orc.fill_dense(SEED, 1, kind, sum(ks), sum(ns))
    Cd = orc.fill_dense(SEED, 2, kind, sum(ms), sum(ns))
    ref = orc.nu_multiply(ms, ns, ks, alpha, Ad, Bd, beta, Cd, *masks)
    return got, orc.nu_scatter(ref, ms, ns, mask=masks[2]), st


@pytest.mark.parametrize("path", ["densified", "blocked"])
@pytest.mark.parametrize("mix", sorted(MIXES))
def test_nu_multiply_matches_oracle(dbm, ctx, orc, path, mix):
    got, ref, st = run_nu(dbm, ctx, orc, mix, path, 0.75, -1.25)
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) <= TOL
    if path == "blocked":
        ms, ns, ks = MIXES[mix]
        assert st["entries"] == len(ms) * len(ns) * len(ks)


@pytest.mark.parametrize("path", ["densified", "blocked"])
@pytest.mark.parametrize("beta", [0.0, -1.25, 1.0])
def test_nu_multiply_integer_bit_exact(dbm, ctx, orc, path, beta):
    got, ref, _ = run_nu(dbm, ctx, orc, "cp2k", path, 0.75, beta, kind=1)
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("m,n,k", [(5, 26, 13), (23, 4, 9), (64, 64, 64), (1, 1, 1), (32, 7, 61), (13, 13, 2)])
def test_mixed_mnk_products(dbm, ctx, orc, m, n, k):
    """§8(f) f4: one (m, n, k) shape per product (LIBCUSMM kernels per (m, n, k)); a grid of
    5 x 3 C blocks of m x n with 4 k-blocks of k, both paths, integer-exact."""
    mix = ([m] * 5, [n] * 3, [k] * 4)
    for path in ("blocked", "densified"):
        got, ref, _ = run_nu(dbm, ctx, orc, mix, path, 0.75, -1.25, kind=1)
        assert np.array_equal(got, ref), (path, m, n, k)


def test_nu_sparse_densified_and_auto(dbm, ctx, orc):
    ms, ns, ks = MIXES["cp2k"]
    masks = (orc.pattern_random(4, 0, len(ms), len(ks), 0.5), orc.pattern_random(4, 1, len(ks), len(ns), 0.5),
             orc.pattern_random(4, 2, len(ms), len(ns), 0.8))
    for path in ("densified", "auto"):
        got, ref, _ = run_nu(dbm, ctx, orc, "cp2k", path, 0.75, -1.25, kind=1, masks=masks)
        assert np.array_equal(got, ref)
    with pytest.raises(dbm.DbmError) as e:
        run_nu(dbm, ctx, orc, "cp2k", "blocked", 0.75, -1.25, masks=masks)
    assert e.value.name == "DBM_ERR_ARG"


def test_nu_alpha_beta_edge_cases(dbm, ctx, orc):
    for path in ("densified", "blocked"):
        got, ref, _ = run_nu(dbm, ctx, orc, "paper", path, 0.0, -1.25, kind=1)
        assert np.array_equal(got, ref)
        got, ref, _ = run_nu(dbm, ctx, orc, "paper", path, 1.0, 0.0, kind=1)
        assert np.array_equal(got, ref)


def test_nu_stacks_equal_uniform_list(dbm, ctx, orc):
    """The stack list is a function of the block structure only (slots, R6/R16): the non-uniform one equals
    the oracle's uniform list for the same block counts."""
    ms, ns, ks = MIXES["cp2k"]
    A, B, C = nu(dbm, ctx, ms, ks), nu(dbm, ctx, ks, ns), nu(dbm, ctx, ms, ns)
    for cap in (30000, 5):
        trip, ptr = dbm.debug_stacks(ctx, A, B, C, 0, cap)
        rtrip, rptr = orc.stacks(len(ms), len(ns), len(ks), cap)
        assert np.array_equal(trip, rtrip) and np.array_equal(ptr, rptr)


def test_nu_partition_validation(dbm, ctx):
    A = nu(dbm, ctx, [5, 7], [3, 4])
    B = nu(dbm, ctx, [4, 3], [6])  # K partition (4, 3) != (3, 4)
    C = nu(dbm, ctx, [5, 7], [6])
    with pytest.raises(dbm.DbmError) as e:
        dbm.multiply(ctx, 1.0, A, B, 0.0, C, "densified")
    assert e.value.name == "DBM_ERR_PARTITION"
    with pytest.raises(dbm.DbmError) as e:
        nu(dbm, ctx, [5, 0], [3])
    assert e.value.name == "DBM_ERR_SHAPE"
    big = nu(dbm, ctx, [65, 3], [2])  # C blocks > 64 rows: the blocked path refuses, densified runs
    Bk = nu(dbm, ctx, [2], [2])
    Ck = nu(dbm, ctx, [65, 3], [2])
    with pytest.raises(dbm.DbmError) as e:
        dbm.multiply(ctx, 1.0, big, Bk, 0.0, Ck, "blocked")
    assert e.value.name == "DBM_ERR_SHAPE"
    dbm.multiply(ctx, 1.0, big, Bk, 0.0, Ck, "densified")


def test_nu_uniform_sizes_are_the_uniform_matrix(dbm, ctx, orc):
    m = nu(dbm, ctx, [22] * 4, [22] * 3)
    assert m.bs == 22 and m.arena_bytes == 4 * 3 * 22 * 22 * 8
    m.fill_random(SEED, 0, 0)
    assert np.array_equal(host(m.arena)[: m.arena_bytes // 8], orc.fill_arena(SEED, 0, 0, 88, 66, 22))


@pytest.mark.parametrize("path", ["densified", "blocked"])
def test_nu_multiply_host_buffers(dbm, ctx, orc, path):
    ms, ns, ks = MIXES["paper"]
    A, B, C = nu(dbm, ctx, ms, ks), nu(dbm, ctx, ks, ns), nu(dbm, ctx, ms, ns)
    hs = []
    for mtx, mid in ((A, 0), (B, 1), (C, 2)):
        mtx.fill_random(SEED, mid, 1)
        h = torch.empty(mtx.arena_bytes // 8, dtype=torch.float64, pin_memory=True)
        mtx.download(h)
        hs.append(h)
    ctx.sync()
    for mtx in (A, B, C):
        mtx.arena.zero_()
    dbm.multiply_host(ctx, 0.75, A, B, -1.25, C, hs[0], hs[1], hs[2], path)
    ctx.sync()
    Ad, Bd, Cd = (orc.fill_dense(SEED, i, 1, r, c) for i, r, c in ((0, sum(ms), sum(ks)), (1, sum(ks), sum(ns)),
                                                                   (2, sum(ms), sum(ns))))
    ref = orc.nu_scatter(orc.nu_multiply(ms, ns, ks, 0.75, Ad, Bd, -1.25, Cd), ms, ns)
    assert np.array_equal(hs[2].numpy(), ref)
