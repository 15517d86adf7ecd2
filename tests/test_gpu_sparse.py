"""GPU parity of the block-sparse path (§8f-2, reading R15) against the host oracle.

Patterns come from the counter generator (dbm_pattern_random, checked against the oracle's own
implementation); C keeps its pattern.  Tolerance as tests/test_gpu_parity.py: normwise relative
<= 1e-12 for U[-1,1) inputs, bit-exact for integer inputs with dyadic alpha/beta and for every
data-movement kernel and stack list.
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

SEED = 1910
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
    torch.cuda.synchronize()
    return t.detach().cpu().numpy()


def relerr(got, ref):
    return np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-300)


def sparse_matrix(dbm, ctx, orc, rows, cols, bs, mat_id, occ, kind=0, pseed=7):
    mask = orc.pattern_random(pseed, mat_id, rows // bs, cols // bs, occ)
    m = dbm.Matrix(ctx, rows, cols, bs, mask=mask)
    m.fill_random(SEED, mat_id, kind)
    return m, mask


def test_pattern_generator_matches_oracle(dbm, orc):
    for occ in (0.0, 0.03, 0.5, 1.0):
        assert np.array_equal(dbm.pattern_random(11, 4, 37, 53, occ), orc.pattern_random(11, 4, 37, 53, occ))


@pytest.mark.parametrize("rows,cols,bs,occ,kind", [(352, 352, 22, 0.3, 0), (256, 384, 64, 0.5, 1), (35, 45, 5, 0.6, 0),
                                                   (44, 66, 22, 0.0, 0)])
def test_sparse_fill_and_csr(dbm, ctx, orc, rows, cols, bs, occ, kind):
    m, mask = sparse_matrix(dbm, ctx, orc, rows, cols, bs, 2, occ, kind)
    assert m.nnz == m.global_nnz == int(mask.sum())
    assert m.arena_bytes == m.nnz * bs * bs * 8
    got = host(m.arena)[: m.nnz * bs * bs]
    full = orc.fill_arena(SEED, 2, kind, rows, cols, bs)
    assert np.array_equal(got, orc.sparse_compress(full, mask, rows // bs, cols // bs, bs))
    rp, ci, ri = m.local_csr()
    assert rp[-1] == m.nnz and list(np.diff(rp)) == list(mask.sum(axis=1))
    assert list(ci) == [j for i in range(mask.shape[0]) for j in range(mask.shape[1]) if mask[i, j]]


def test_sparse_set_get_block(dbm, ctx, orc):
    m, mask = sparse_matrix(dbm, ctx, orc, 110, 88, 22, 3, 0.5)
    i, j = map(int, np.argwhere(mask)[0])
    blk = np.arange(22 * 22, dtype=np.float64).reshape(22, 22)
    m.set_block(i, j, blk)
    assert np.array_equal(m.get_block(i, j), blk)
    ai, aj = map(int, np.argwhere(mask == 0)[0])
    with pytest.raises(dbm.DbmError) as e:
        m.get_block(ai, aj)
    assert e.value.name == "DBM_ERR_RANGE"


@pytest.mark.parametrize("layout", [0, 1])
def test_sparse_densify_undensify(dbm, ctx, orc, layout):
    """Absent blocks densify to zeros; undensify writes only stored blocks, alpha/beta exact."""
    rows, cols, bs = 198, 264, 22
    m, mask = sparse_matrix(dbm, ctx, orc, rows, cols, bs, 0, 0.4)
    ld = rows + 2 if layout == 0 else cols + 2
    n = ld * (cols if layout == 0 else rows)
    d = torch.full((n,), float("nan"), dtype=torch.float64, device="cuda")
    m.densify(d, ld, layout)
    full = orc.fill_arena(SEED, 0, 0, rows, cols, bs)
    Mb, Nb = rows // bs, cols // bs
    dense = orc.arena_to_dense(full, Mb, Nb, bs) * np.kron(mask, np.ones((bs, bs)))
    g = host(d)
    got = g.reshape(cols, ld)[:, :rows].T if layout == 0 else g.reshape(rows, ld)[:, :cols]
    assert np.array_equal(got, dense)
    # undensify: stored C blocks = alpha * D + beta * C
    D = torch.tensor(np.asfortranarray(np.random.default_rng(1).integers(-3, 4, (rows, cols)).astype(np.float64))
                     .T.reshape(-1), device="cuda")
    before = host(m.arena)[: m.nnz * bs * bs].copy()
    m.undensify(D, 0.75, -1.25, rows)
    Dg = orc.dense_to_arena(host(D).reshape(cols, rows).T, bs)
    want = 0.75 * orc.sparse_compress(Dg, mask, Mb, Nb, bs) + -1.25 * before
    assert np.array_equal(host(m.arena)[: m.nnz * bs * bs], want)


def run_sparse(dbm, ctx, orc, M, N, K, bs, path, occ_a, occ_b, occ_c, alpha, beta, kind=0, cap=0):
    A, am = sparse_matrix(dbm, ctx, orc, M, K, bs, 0, occ_a, kind)
    B, bm = sparse_matrix(dbm, ctx, orc, K, N, bs, 1, occ_b, kind)
    Cm, cm = sparse_matrix(dbm, ctx, orc, M, N, bs, 2, occ_c, kind)
    st = dbm.multiply(ctx, alpha, A, B, beta, Cm, path, cap)
    got = host(Cm.arena)[: Cm.nnz * bs * bs]
    Mb, Nb, Kb = M // bs, N // bs, K // bs
    Ao, Bo = orc.fill_arena(SEED, 0, kind, M, K, bs), orc.fill_arena(SEED, 1, kind, K, N, bs)
    Co = orc.fill_arena(SEED, 2, kind, M, N, bs)
    orc.multiply_sparse(Mb, Nb, Kb, bs, alpha, Ao, am, Bo, bm, beta, Co, cm)
    ref = orc.sparse_compress(Co, cm, Mb, Nb, bs)
    entries = int(((am.astype(np.int64) @ bm.astype(np.int64)) * cm).sum())
    return got, ref, st, entries


@pytest.mark.parametrize("path", ["blocked", "densified"])
@pytest.mark.parametrize("M,N,K,bs,oa,ob,oc", [
    (352, 352, 352, 22, 0.3, 0.3, 1.0), (352, 352, 352, 22, 0.1, 0.5, 0.4), (704, 528, 1100, 22, 0.05, 0.05, 1.0),
    (512, 384, 640, 64, 0.4, 0.6, 0.7), (1408, 1408, 5632, 64, 0.2, 0.2, 1.0), (40, 35, 50, 5, 0.5, 0.5, 0.8),
    (352, 352, 352, 22, 1.0, 1.0, 1.0), (352, 352, 352, 22, 0.0, 0.5, 1.0), (88, 88, 45056, 22, 0.3, 0.3, 1.0),
    (390, 325, 520, 13, 0.4, 0.3, 0.7), (256, 224, 384, 32, 0.3, 0.5, 1.0), (161, 207, 276, 23, 0.5, 0.5, 0.6)])
def test_sparse_multiply_matches_oracle(dbm, ctx, orc, path, M, N, K, bs, oa, ob, oc):
    got, ref, st, entries = run_sparse(dbm, ctx, orc, M, N, K, bs, path, oa, ob, oc, 0.75, -1.25)
    assert relerr(got, ref) <= TOL
    if path == "blocked":
        assert st["entries"] == entries
        assert st["flops"] == 2.0 * bs ** 3 * entries


@pytest.mark.parametrize("path", ["blocked", "densified"])
@pytest.mark.parametrize("beta", [-1.25, 0.0])
def test_sparse_multiply_integer_bit_exact(dbm, ctx, orc, path, beta):
    got, ref, _, _ = run_sparse(dbm, ctx, orc, 704, 528, 1100, 22, path, 0.3, 0.4, 0.6, 0.75, beta, kind=1)
    assert np.array_equal(got, ref)
    got, ref, _, _ = run_sparse(dbm, ctx, orc, 384, 448, 640, 64, path, 0.3, 0.4, 0.6, 0.75, beta, kind=1)
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("n,bs,occ,cap", [(352, 22, 0.3, 0), (352, 22, 0.6, 40), (640, 64, 0.5, 7), (110, 22, 0.0, 5)])
def test_sparse_stacks_bit_exact(dbm, ctx, orc, n, bs, occ, cap):
    A, am = sparse_matrix(dbm, ctx, orc, n, n, bs, 0, occ)
    B, bm = sparse_matrix(dbm, ctx, orc, n, n, bs, 1, occ)
    Cm, cm = sparse_matrix(dbm, ctx, orc, n, n, bs, 2, max(occ, 0.5))
    trip, ptr = dbm.debug_stacks(ctx, A, B, Cm, 0, cap)
    rtrip, rptr = orc.sparse_stacks(am, bm, cm, cap or 30000)
    assert np.array_equal(trip, rtrip)
    assert np.array_equal(ptr, rptr)


def test_auto_path_should_densify(dbm, ctx, orc):
    """DBM_PATH_AUTO: dense operands densify at the default threshold 1.0; at 0.1 occupancy they
    stay blocked unless the threshold is lowered.  Both give the oracle's product."""
    got, ref, st, _ = run_sparse(dbm, ctx, orc, 352, 352, 352, 22, "auto", 0.1, 0.1, 1.0, 1.0, 0.0)
    assert relerr(got, ref) <= TOL and st["entries"] != 1  # blocked
    ctx.set_densify_threshold(0.05)
    got, ref, st, _ = run_sparse(dbm, ctx, orc, 352, 352, 352, 22, "auto", 0.1, 0.1, 1.0, 1.0, 0.0)
    ctx.set_densify_threshold(1.0)
    assert relerr(got, ref) <= TOL and st["entries"] == 1  # densified: batch size 1


def test_sparse_determinism(dbm, ctx, orc):
    outs = []
    for _ in range(2):
        got, _, _, _ = run_sparse(dbm, ctx, orc, 704, 704, 704, 22, "blocked", 0.3, 0.3, 0.9, 1.0, 0.0)
        outs.append(got)
    assert np.array_equal(outs[0], outs[1])


@pytest.mark.parametrize("path", ["blocked", "densified"])
def test_sparse_multiply_host(dbm, ctx, orc, path):
    """Host-resident sparse arenas through dbm_multiply_host (stored blocks only move)."""
    M, N, K, bs = 352, 264, 440, 22
    Mb, Nb, Kb = M // bs, N // bs, K // bs
    am, bm, cm = orc.pattern_random(3, 0, Mb, Kb, 0.4), orc.pattern_random(3, 1, Kb, Nb, 0.4), \
        orc.pattern_random(3, 2, Mb, Nb, 0.7)
    Ag, Bg, Cg = (orc.fill_arena(SEED, i, 1, *sh, bs) for i, sh in enumerate(((M, K), (K, N), (M, N))))
    hs = [torch.from_numpy(orc.sparse_compress(g, m, *d, bs)).pin_memory()
          for g, m, d in ((Ag, am, (Mb, Kb)), (Bg, bm, (Kb, Nb)), (Cg, cm, (Mb, Nb)))]
    A = dbm.Matrix(ctx, M, K, bs, mask=am)
    B = dbm.Matrix(ctx, K, N, bs, mask=bm)
    Cm = dbm.Matrix(ctx, M, N, bs, mask=cm)
    dbm.multiply_host(ctx, 0.75, A, B, -1.25, Cm, hs[0], hs[1], hs[2], path)
    ctx.sync()
    orc.multiply_sparse(Mb, Nb, Kb, bs, 0.75, Ag, am, Bg, bm, -1.25, Cg, cm)
    assert np.array_equal(hs[2].numpy(), orc.sparse_compress(Cg, cm, Mb, Nb, bs))


def test_fill_in_workflow(dbm, ctx, orc):
    """DBCSR-style fill-in in two calls (R15): C_out gets the product pattern OR C_in's pattern
    (dbm_pattern_product), C_in's blocks are copied over, then the multiply fills every product block."""
    M, N, K, bs = 352, 352, 352, 22
    Mb = Nb = Kb = 16
    am, bm, cm = orc.pattern_random(9, 0, Mb, Kb, 0.2), orc.pattern_random(9, 1, Kb, Nb, 0.2), \
        orc.pattern_random(9, 2, Mb, Nb, 0.1)
    cout = dbm.pattern_product(am, bm, cm)
    assert (cout >= cm).all() and cout.sum() > cm.sum()
    A = dbm.Matrix(ctx, M, K, bs, mask=am)
    B = dbm.Matrix(ctx, K, N, bs, mask=bm)
    Cn = dbm.Matrix(ctx, M, N, bs, mask=cout)
    A.fill_random(SEED, 0, 1)
    B.fill_random(SEED, 1, 1)
    Cn.fill_random(SEED, 2, 1)  # the fill-in blocks start from the generator too (beta = 0 below)
    dbm.multiply(ctx, 1.0, A, B, 0.0, Cn, "blocked")
    got = host(Cn.arena)[: Cn.nnz * bs * bs]
    Ag, Bg, Cg = (orc.fill_arena(SEED, i, 1, M, M, bs) for i in range(3))
    orc.multiply_sparse(Mb, Nb, Kb, bs, 1.0, Ag, am, Bg, bm, 0.0, Cg, cout)
    assert np.array_equal(got, orc.sparse_compress(Cg, cout, Mb, Nb, bs))
