"""GPU parity: the CUDA path (through the C ABI) against the host oracle, element by element.

Tolerance (north star): normwise relative Frobenius error <= 1e-12 for U[-1,1) inputs; bit-exact
for integer inputs with dyadic alpha/beta, for every data-movement kernel (fill, densify,
undensify) and for stack lists.  Single GPU (grid 1x1); the multi-rank path is in
tests/test_multigpu.py.
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


def host(t: torch.Tensor) -> np.ndarray:
    torch.cuda.synchronize()
    return t.detach().cpu().numpy()


def relerr(got, ref):
    return np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-300)


# ------------------------------------------------------------------ data movement (bit-exact)
@pytest.mark.parametrize("rows,cols,bs,kind", [(352, 352, 22, 0), (128, 192, 64, 1), (15, 21, 3, 0), (0, 44, 22, 0)])
def test_fill_bit_exact(dbm, ctx, orc, rows, cols, bs, kind):
    m = dbm.Matrix(ctx, rows, cols, bs)
    m.fill_random(SEED, 2, kind)
    got = host(m.arena)[: m.arena_bytes // 8]
    assert np.array_equal(got, orc.fill_arena(SEED, 2, kind, rows, cols, bs))


def test_set_get_block_and_ownership(dbm, ctx):
    m = dbm.Matrix(ctx, 66, 44, 22)
    blk = np.arange(22 * 22, dtype=np.float64).reshape(22, 22)
    m.set_block(2, 1, blk)
    assert np.array_equal(m.get_block(2, 1), blk)
    with pytest.raises(dbm.DbmError) as e:
        m.get_block(3, 0)
    assert e.value.name == "DBM_ERR_RANGE"
    assert m.owner_of_block(2, 1) == 0
    rp, ci, ri = m.local_csr()
    assert list(rp) == [0, 2, 4, 6] and list(ci) == [0, 1] * 3 and list(ri) == [0, 1, 2]


@pytest.mark.parametrize("rows,cols,bs", [(352, 352, 22), (128, 320, 64), (21, 15, 3), (198, 374, 22)])
@pytest.mark.parametrize("layout", [0, 1])
@pytest.mark.parametrize("pad", [0, 3, 4])  # even ld takes the vectorised fast path for bs 22 / 64
def test_densify_bit_exact(dbm, ctx, orc, rows, cols, bs, layout, pad):
    m = dbm.Matrix(ctx, rows, cols, bs)
    m.fill_random(SEED, 0, 0)
    mloc, nloc = rows // bs, cols // bs
    ld = (mloc * bs + pad) if layout == 0 else (nloc * bs + pad)  # padded leading dimension
    n = ld * (nloc * bs if layout == 0 else mloc * bs)
    d = torch.full((n,), float("nan"), dtype=torch.float64, device="cuda")
    m.densify(d, ld, layout)
    got = host(d)
    arena = orc.fill_arena(SEED, 0, 0, rows, cols, bs)
    ref = orc.densify_cols(arena, mloc, nloc, bs, np.arange(nloc), layout)
    if layout == 0:
        got = got.reshape(nloc * bs, ld)[:, : mloc * bs]
        ref = ref.reshape(nloc * bs, mloc * bs)
    else:
        got = got.reshape(mloc * bs, ld)[:, : nloc * bs]
        ref = ref.reshape(mloc * bs, nloc * bs)
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("alpha,beta", [(1.0, 0.0), (0.75, -1.25), (-2.5, 1.0)])
def test_undensify_bit_exact(dbm, ctx, orc, alpha, beta):
    rows, cols, bs = 352, 264, 22
    m = dbm.Matrix(ctx, rows, cols, bs)
    m.fill_random(SEED, 2, 0)
    if beta == 0.0:
        m.arena.fill_(float("nan"))  # beta == 0 must not read C
    dense = torch.rand(rows * cols, dtype=torch.float64, device="cuda") * 2 - 1
    m.undensify(dense, alpha, beta)
    arena = orc.fill_arena(SEED, 2, 0, rows, cols, bs)
    orc.undensify(host(dense), rows, rows // bs, cols // bs, bs, alpha, beta, arena)
    assert np.array_equal(host(m.arena)[: arena.size], arena)


# ------------------------------------------------------------------ dense FP64 GEMM kernel
@pytest.mark.parametrize("M,N,K,splitk", [(128, 128, 16, 1), (352, 352, 352, 1), (200, 136, 50, 1),
                                          (1, 1, 1, 1), (257, 129, 1000, 1), (300, 200, 4096, 3),
                                          (128, 64, 0, 1), (704, 384, 7936, 0)])
def test_dgemm_kernel(dbm, ctx, M, N, K, splitk):
    g = torch.Generator().manual_seed(M * 7 + N * 3 + K)
    lda = ldb = K + (K % 2) + 2
    At = torch.rand(M, lda, dtype=torch.float64, generator=g) * 2 - 1
    Bt = torch.rand(N, ldb, dtype=torch.float64, generator=g) * 2 - 1
    Cc = torch.rand(N, M, dtype=torch.float64, generator=g) * 2 - 1  # column-major C (ldc = M)
    alpha, beta = 0.75, -1.25
    ref = alpha * (At[:, :K].numpy() @ Bt[:, :K].numpy().T) + beta * Cc.numpy().T
    dA, dB, dC = At.cuda(), Bt.cuda(), Cc.cuda()
    part = torch.empty(max(splitk, 64) * M * N + 1, dtype=torch.float64, device="cuda")
    dbm.debug_dgemm(ctx, M, N, K, alpha, dA, lda, dB, ldb, beta, dC, M, splitk, part)
    got = host(dC).T
    assert relerr(got, ref) <= TOL
    assert np.abs(got - ref).max() <= 1e-13 * max(K, 1)


def test_dgemm_integer_exact(dbm, ctx):
    M, N, K = 333, 190, 2048
    g = torch.Generator().manual_seed(5)
    At = torch.randint(-2, 3, (M, K), generator=g).double()
    Bt = torch.randint(-2, 3, (N, K), generator=g).double()
    Cc = torch.randint(-2, 3, (N, M), generator=g).double()
    ref = 0.75 * (At.numpy() @ Bt.numpy().T) - 1.25 * Cc.numpy().T
    for splitk in (1, 4):
        dC = Cc.cuda()
        part = torch.empty(splitk * M * N + 1, dtype=torch.float64, device="cuda")
        dbm.debug_dgemm(ctx, M, N, K, 0.75, At.cuda(), K, Bt.cuda(), K, -1.25, dC, M, splitk, part)
        assert np.array_equal(host(dC).T, ref)


# ------------------------------------------------------------------ stacks (bit-exact)
@pytest.mark.parametrize("n,bs,cap", [(352, 22, 30000), (352, 22, 100), (352, 22, 7), (640, 64, 30), (0, 22, 10)])
def test_stacks_bit_exact(dbm, ctx, orc, n, bs, cap):
    A, B, C = (dbm.Matrix(ctx, n, n, bs) for _ in range(3))
    trip, ptr = dbm.debug_stacks(ctx, A, B, C, 0, cap)
    nb = n // bs
    rtrip, rptr = orc.stacks(nb, nb, nb, cap)
    assert np.array_equal(trip, rtrip)
    assert np.array_equal(ptr, rptr)


@pytest.mark.parametrize("Mb,Nb,Kb,bs,cap", [(13, 7, 29, 22, 7), (13, 7, 29, 22, 100), (7, 13, 29, 22, 30000),
                                           (5, 9, 3, 64, 4), (1, 11, 40, 22, 30), (9, 1, 2, 5, 3)])
def test_stacks_bit_exact_non_square(dbm, ctx, orc, Mb, Nb, Kb, bs, cap):
    """Stack lists on rectangular local grids (mloc != nloc, the bisection splits the longer side) and
    runs longer than the cap (kb > cap splits a run into ceil(kb/cap) stacks)."""
    A, B, C = dbm.Matrix(ctx, Mb * bs, Kb * bs, bs), dbm.Matrix(ctx, Kb * bs, Nb * bs, bs), dbm.Matrix(ctx, Mb * bs, Nb * bs, bs)
    trip, ptr = dbm.debug_stacks(ctx, A, B, C, 0, cap)
    rtrip, rptr = orc.stacks(Mb, Nb, Kb, cap)
    assert np.array_equal(trip, rtrip)
    assert np.array_equal(ptr, rptr)


# ------------------------------------------------------------------ pack panel (a3, bit-exact)
@pytest.mark.parametrize("rows,cols,bs", [(352, 616, 22), (320, 448, 64), (65, 91, 13), (30, 45, 5)])
@pytest.mark.parametrize("operand", [0, 1])
@pytest.mark.parametrize("first,stride", [(0, 1), (1, 2), (0, 4), (2, 3)])
def test_pack_panel_bit_exact(dbm, ctx, orc, rows, cols, bs, operand, first, stride):
    """a3: the GPU panel pack (dbm_debug_pack_panel) against orc_pack_panel (brute-force pinned in
    test_oracle_pins.py::test_pack_panel_brute_force), every block size alignment (bs^2 odd: blocks
    alternate 8 mod 16 bytes)."""
    m = dbm.Matrix(ctx, rows, cols, bs)
    m.fill_random(SEED, operand, 0)
    mloc, nloc = rows // bs, cols // bs
    lim = nloc if operand == 0 else mloc
    nk = max(0, (lim - 1 - first) // stride + 1)
    kidx = [first + q * stride for q in range(nk)]
    other = mloc if operand == 0 else nloc
    out = torch.full((max(other * nk * bs * bs, 1),), float("nan"), dtype=torch.float64, device="cuda")
    dbm.debug_pack_panel(m, operand, first, stride, nk, out)
    ref = orc.pack_panel(orc.fill_arena(SEED, operand, 0, rows, cols, bs), mloc, nloc, bs, operand, kidx)
    assert np.array_equal(host(out)[: ref.size], ref)


@pytest.mark.parametrize("bs", [22, 13])
def test_pack_panel_chunks_with_pitch(dbm, ctx, orc, bs):
    """The host pipeline packs an A panel K-chunk by K-chunk at the panel's pitch: chunks [q0, q1) packed
    into columns q0.. of every packed row must assemble the whole panel."""
    rows, cols = 10 * bs, 17 * bs
    m = dbm.Matrix(ctx, rows, cols, bs)
    m.fill_random(SEED, 0, 1)
    mloc, nloc = 10, 17
    first, stride = 1, 2
    kb = (nloc - 1 - first) // stride + 1
    bb = bs * bs
    out = torch.full((mloc * kb * bb,), float("nan"), dtype=torch.float64, device="cuda")
    bounds = [0, 0, 1, 2, 5, kb]
    for q0, q1 in zip(bounds[:-1], bounds[1:]):
        if q1 > q0:
            dbm.debug_pack_panel(m, 0, first + q0 * stride, stride, q1 - q0, out[q0 * bb:], pitch=kb)
    ref = orc.pack_panel(orc.fill_arena(SEED, 0, 1, rows, cols, bs), mloc, nloc, bs, 0,
                         [first + q * stride for q in range(kb)])
    assert np.array_equal(host(out), ref)


def test_pack_panel_validation(dbm, ctx):
    m = dbm.Matrix(ctx, 88, 66, 22)
    out = torch.empty(64 * 22 * 22, dtype=torch.float64, device="cuda")
    for args, name in [((2, 0, 1, 1), "DBM_ERR_ARG"), ((0, 2, 1, 2), "DBM_ERR_RANGE"), ((1, 0, 1, 5), "DBM_ERR_RANGE"),
                       ((0, 0, 0, 1), "DBM_ERR_ARG")]:
        with pytest.raises(dbm.DbmError) as e:
            dbm.debug_pack_panel(m, *args, out)
        assert e.value.name == name


# ------------------------------------------------------------------ full multiply vs the oracle
def run_multiply(dbm, ctx, orc, M, N, K, bs, path, alpha, beta, kind=0, cap=0, chunk=None):
    A, B, C = dbm.Matrix(ctx, M, K, bs), dbm.Matrix(ctx, K, N, bs), dbm.Matrix(ctx, M, N, bs)
    A.fill_random(SEED, 0, kind)
    B.fill_random(SEED, 1, kind)
    C.fill_random(SEED, 2, kind)
    if chunk is not None:
        ctx.set_dense_chunk_bytes(chunk)
    st = dbm.multiply(ctx, alpha, A, B, beta, C, path, cap)
    if chunk is not None:
        ctx.set_dense_chunk_bytes(16 << 30)
    got = host(C.arena)[: C.arena_bytes // 8]
    Ao, Bo = orc.fill_arena(SEED, 0, kind, M, K, bs), orc.fill_arena(SEED, 1, kind, K, N, bs)
    Co = orc.fill_arena(SEED, 2, kind, M, N, bs)
    orc.multiply_blocked(M // bs, N // bs, K // bs, bs, alpha, Ao, Bo, beta, Co)
    return got, Co, st


@pytest.mark.parametrize("path", ["densified", "blocked"])
@pytest.mark.parametrize("M,N,K,bs", [(352, 352, 352, 22), (128, 192, 256, 64), (66, 110, 44, 22),
                                      (110, 154, 66, 22), (154, 330, 198, 22), (320, 192, 448, 64),
                                      (1408, 704, 2816, 64), (2816, 2816, 2816, 22), (12, 21, 30, 3), (256, 192, 320, 4),
                                      (88, 88, 90112, 22), (154, 110, 45034, 22),   # few long runs: smm split-K
                                      (128, 192, 16384, 64), (320, 64, 12800, 64)])
def test_multiply_matches_oracle(dbm, ctx, orc, path, M, N, K, bs):
    got, ref, st = run_multiply(dbm, ctx, orc, M, N, K, bs, path, 0.75, -1.25)
    assert relerr(got, ref) <= TOL
    if path == "densified":
        assert st["entries"] == st["stacks"] == 1  # P:198 batch size 1
    else:
        nb = (M // bs) * (N // bs) * (K // bs)
        assert st["entries"] == nb


@pytest.mark.parametrize("path", ["densified", "blocked"])
def test_multiply_integer_bit_exact(dbm, ctx, orc, path):
    got, ref, _ = run_multiply(dbm, ctx, orc, 704, 528, 1100, 22, path, 0.75, -1.25, kind=1)
    assert np.array_equal(got, ref)
    # 32 x 32 blocks: the bisection visits 4 x 4 squares -> the unpadded 88 x 88 bs-22 kernel
    got, ref, _ = run_multiply(dbm, ctx, orc, 704, 704, 1100, 22, path, 0.75, -1.25, kind=1)
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("nb,kb", [(8, 1), (8, 2), (8, 3), (8, 5), (8, 6), (8, 7), (8, 8), (8, 9), (8, 17),
                                   (64, 9), (64, 6), (32, 40)])
@pytest.mark.parametrize("beta", [0.0, -1.25])
def test_smm22q_item_lengths(dbm, ctx, orc, nb, kb, beta):
    """The 4 x 4-square bs-22 kernel over every item regime: 1..9 stages of 2 k-blocks (items shorter
    than STAGES + 1 keep the CTA barriers, longer ones run with double-buffered destinations), odd kb
    (a predicated half stage at the end), and 256 squares (several items per CTA).  Integer inputs: exact."""
    n = nb * 22
    got, ref, st = run_multiply(dbm, ctx, orc, n, n, kb * 22, 22, "blocked", 0.75, beta, kind=1)
    assert np.array_equal(got, ref)
    assert st["entries"] == nb * nb * kb


@pytest.mark.parametrize("bs", [4, 5, 6, 7, 8, 9, 13, 16, 23, 26, 32])
def test_blocked_small_block_sizes(dbm, ctx, orc, bs):
    """The per-size DMMA run kernels (bs 4..32 except 22 / 64; bs 7 stays on the FMA kernel) on uniform runs:
    odd block sizes take the 8-byte staging branch, bs 26 / 32 the 4-warp teams; beta 0 and beta != 0."""
    for (mb, nb, kb), beta in [((7, 5, 9), -1.25), ((40, 36, 3), 0.0), ((3, 2, 61), 1.0)]:
        got, ref, st = run_multiply(dbm, ctx, orc, mb * bs, nb * bs, kb * bs, bs, "blocked", 0.75, beta)
        assert relerr(got, ref) <= TOL
        assert st["entries"] == mb * nb * kb
    got, ref, _ = run_multiply(dbm, ctx, orc, 9 * bs, 11 * bs, 13 * bs, bs, "blocked", 0.75, -1.25, kind=1)
    assert np.array_equal(got, ref)


def test_densified_k_chunking(dbm, ctx, orc):
    """Single-rank K-chunked densify -> GEMM accumulate (how 63,360^3 fits HBM) equals the oracle."""
    M = N = 384
    K, bs = 1280, 64
    chunk = (M + N) * bs * 8 * 3  # 3 block columns per chunk -> 7 chunks, the last ragged
    got, ref, st = run_multiply(dbm, ctx, orc, M, N, K, bs, "densified", 0.75, -1.25, chunk=chunk)
    assert st["gemm_launches"] == 7
    assert relerr(got, ref) <= TOL
    got, ref, _ = run_multiply(dbm, ctx, orc, M, N, K, bs, "densified", 0.75, -1.25, kind=1, chunk=chunk)
    assert np.array_equal(got, ref)


def test_identity_and_permutation_routing(dbm, ctx, orc):
    """A = permutation: C must be an exact row permutation of B (any misrouted block shows)."""
    n, bs = 352, 22
    rng = np.random.default_rng(1)
    perm = rng.permutation(n)
    P = np.eye(n)[perm]
    for path in ("densified", "blocked"):
        A, B, C = dbm.Matrix(ctx, n, n, bs), dbm.Matrix(ctx, n, n, bs), dbm.Matrix(ctx, n, n, bs)
        A.arena[: n * n].copy_(torch.from_numpy(orc.dense_to_arena(P, bs)))
        B.fill_random(SEED, 1, 0)
        dbm.multiply(ctx, 1.0, A, B, 0.0, C, path)
        got = orc.arena_to_dense(host(C.arena)[: n * n], n // bs, n // bs, bs)
        Bd = orc.arena_to_dense(orc.fill_arena(SEED, 1, 0, n, n, bs), n // bs, n // bs, bs)
        assert np.array_equal(got, Bd[perm])


def test_alpha_beta_edge_cases(dbm, ctx, orc):
    n, bs = 176, 22
    for path in ("densified", "blocked"):
        A, B, C = dbm.Matrix(ctx, n, n, bs), dbm.Matrix(ctx, n, n, bs), dbm.Matrix(ctx, n, n, bs)
        # alpha == 0: A and B are not read; C = beta*C exactly
        A.arena.fill_(float("nan"))
        B.arena.fill_(float("nan"))
        C.fill_random(SEED, 2, 0)
        dbm.multiply(ctx, 0.0, A, B, -1.25, C, path)
        assert np.array_equal(host(C.arena), -1.25 * orc.fill_arena(SEED, 2, 0, n, n, bs))
        # beta == 0: C is not read (NaN stays out)
        A.fill_random(SEED, 0, 0)
        B.fill_random(SEED, 1, 0)
        C.arena.fill_(float("nan"))
        dbm.multiply(ctx, 1.0, A, B, 0.0, C, path)
        assert not torch.isnan(C.arena).any().item()


def test_empty_and_degenerate_shapes(dbm, ctx, orc):
    for path in ("densified", "blocked"):
        # K = 0: C = beta*C
        A, B, C = dbm.Matrix(ctx, 44, 0, 22), dbm.Matrix(ctx, 0, 66, 22), dbm.Matrix(ctx, 44, 66, 22)
        C.fill_random(SEED, 2, 0)
        dbm.multiply(ctx, 1.0, A, B, 0.5, C, path)
        assert np.array_equal(host(C.arena), 0.5 * orc.fill_arena(SEED, 2, 0, 44, 66, 22))
        # M = 0
        A, B, C = dbm.Matrix(ctx, 0, 44, 22), dbm.Matrix(ctx, 44, 66, 22), dbm.Matrix(ctx, 0, 66, 22)
        dbm.multiply(ctx, 1.0, A, B, 0.0, C, path)
        torch.cuda.synchronize()
        # single block
        got, ref, _ = run_multiply(dbm, ctx, orc, 22, 22, 22, 22, path, 0.75, -1.25)
        assert relerr(got, ref) <= TOL


def test_validation_errors_leave_c_untouched(dbm, ctx):
    A, B, C = dbm.Matrix(ctx, 44, 66, 22), dbm.Matrix(ctx, 44, 66, 22), dbm.Matrix(ctx, 44, 66, 22)
    C.arena.fill_(3.0)
    with pytest.raises(dbm.DbmError) as e:
        dbm.multiply(ctx, 1.0, A, B, 0.0, C)
    assert e.value.name == "DBM_ERR_SHAPE"
    B2 = dbm.Matrix(ctx, 66, 66, 22)
    with pytest.raises(dbm.DbmError) as e:
        dbm.multiply(ctx, 1.0, A, B2, 0.0, A)
    assert e.value.name == "DBM_ERR_ALIAS"
    B3 = dbm.Matrix(ctx, 66, 66, 33)
    with pytest.raises(dbm.DbmError) as e:
        dbm.multiply(ctx, 1.0, A, B3, 0.0, C)
    assert e.value.name in ("DBM_ERR_PARTITION", "DBM_ERR_SHAPE")
    with pytest.raises(dbm.DbmError) as e:
        dbm.Matrix(ctx, 45, 44, 22)
    assert e.value.name == "DBM_ERR_SHAPE"
    torch.cuda.synchronize()
    assert (C.arena == 3.0).all().item()


def test_determinism(dbm, ctx):
    n, bs = 1408, 64
    outs = []
    for _ in range(2):
        A, B, C = dbm.Matrix(ctx, n, n, bs), dbm.Matrix(ctx, n, n, bs), dbm.Matrix(ctx, n, n, bs)
        A.fill_random(SEED, 0, 0)
        B.fill_random(SEED, 1, 0)
        C.fill_random(SEED, 2, 0)
        dbm.multiply(ctx, 0.75, A, B, -1.25, C, "densified")
        outs.append(host(C.arena).copy())
    assert np.array_equal(outs[0], outs[1])


def test_blocked_vs_densified_agree(dbm, ctx, orc):
    a, _, _ = run_multiply(dbm, ctx, orc, 704, 704, 704, 22, "blocked", 1.0, 0.0)
    b, ref, _ = run_multiply(dbm, ctx, orc, 704, 704, 704, 22, "densified", 1.0, 0.0)
    assert relerr(a, b) <= 2 * TOL


def test_host_upload_download_roundtrip(dbm, ctx, orc):
    m = dbm.Matrix(ctx, 352, 264, 22)
    x = torch.from_numpy(orc.fill_arena(SEED, 0, 0, 352, 264, 22))
    m.upload(x)  # pageable: staged through the pinned double buffer
    y = torch.empty_like(x)
    m.download(y)
    assert torch.equal(x, y)
    xp = x.pin_memory()
    m.upload(xp)
    yp = torch.empty_like(x).pin_memory()
    m.download(yp)
    ctx.sync()
    assert torch.equal(x, yp)


@pytest.mark.parametrize("path,pinned,chunk", [("densified", True, 3), ("densified", True, None),
                                               ("blocked", True, None), ("densified", False, None)])
def test_multiply_host_streamed(dbm, ctx, orc, path, pinned, chunk):
    """dbm_multiply_host (P:25 host-resident matrices, P:174 double buffering): A and B stream from
    host memory (K-chunk by K-chunk on the single-rank densified path), C comes back to the host."""
    M, N, K, bs = 384, 320, 1280, 64
    Ah = torch.from_numpy(orc.fill_arena(SEED, 0, 0, M, K, bs))
    Bh = torch.from_numpy(orc.fill_arena(SEED, 1, 0, K, N, bs))
    Ch = torch.from_numpy(orc.fill_arena(SEED, 2, 0, M, N, bs))
    if pinned:
        Ah, Bh, Ch = Ah.pin_memory(), Bh.pin_memory(), Ch.pin_memory()
    A, B, C = dbm.Matrix(ctx, M, K, bs), dbm.Matrix(ctx, K, N, bs), dbm.Matrix(ctx, M, N, bs)
    if chunk is not None:
        ctx.set_dense_chunk_bytes((M + N) * bs * 8 * chunk)
    dbm.multiply_host(ctx, 0.75, A, B, -1.25, C, Ah, Bh, Ch, path)
    ctx.sync()
    if chunk is not None:
        ctx.set_dense_chunk_bytes(16 << 30)
    ref = orc.fill_arena(SEED, 2, 0, M, N, bs)
    orc.multiply_blocked(M // bs, N // bs, K // bs, bs, 0.75, orc.fill_arena(SEED, 0, 0, M, K, bs),
                         orc.fill_arena(SEED, 1, 0, K, N, bs), -1.25, ref)
    assert relerr(Ch.numpy(), ref) <= TOL


@pytest.mark.parametrize("kind", [0, 1])
def test_multiply_host_row_panels(dbm, ctx, orc, kind):
    """Enough block rows (>= 8) that the last GEMM chunk runs in row panels whose undensify + download
    overlap the next panel, with geometric upload chunks; beta != 0 reads C_host."""
    M, N, K, bs = 704, 352, 1100, 22
    hs = [torch.from_numpy(orc.fill_arena(SEED, i, kind, *sh, bs)).pin_memory()
          for i, sh in enumerate(((M, K), (K, N), (M, N)))]
    A, B, C = dbm.Matrix(ctx, M, K, bs), dbm.Matrix(ctx, K, N, bs), dbm.Matrix(ctx, M, N, bs)
    ctx.set_dense_chunk_bytes((M + N) * bs * 8 * 7)
    dbm.multiply_host(ctx, 0.75, A, B, -1.25, C, hs[0], hs[1], hs[2], "densified")
    ctx.sync()
    ctx.set_dense_chunk_bytes(16 << 30)
    ref = orc.fill_arena(SEED, 2, kind, M, N, bs)
    orc.multiply_blocked(M // bs, N // bs, K // bs, bs, 0.75, orc.fill_arena(SEED, 0, kind, M, K, bs),
                         orc.fill_arena(SEED, 1, kind, K, N, bs), -1.25, ref)
    if kind == 1:
        assert np.array_equal(hs[2].numpy(), ref)
    else:
        assert relerr(hs[2].numpy(), ref) <= TOL


@pytest.mark.parametrize("path", ["densified", "blocked"])
def test_multiply_timing_fields(dbm, ctx, path):
    """dbm_multiply_timing (the dbm_stats ms_* fields): the call's device time and its phases;
    the phases fit inside the call (kernels of one stream), the exposed remainder is what is left."""
    A, B, C = dbm.Matrix(ctx, 704, 704, 22), dbm.Matrix(ctx, 704, 704, 22), dbm.Matrix(ctx, 704, 704, 22)
    for m, i in ((A, 0), (B, 1), (C, 2)):
        m.fill_random(SEED, i, 0)
    ctx.set_profiling(True)
    dbm.multiply(ctx, 1.0, A, B, 0.0, C, path)
    t = ctx.multiply_timing()
    ctx.set_profiling(False)
    for k in range(6):
        ctx.profile_read(k)
    assert t["ms_total"] > 0 and t["ms_local"] > 0
    assert t["ms_densify"] + t["ms_local"] + t["ms_undensify"] <= t["ms_total"] * 1.001 + 1e-3
    assert t["ms_comm_exposed"] >= 0
    if path == "densified":
        assert t["ms_densify"] > 0 and t["ms_undensify"] > 0
    with pytest.raises(dbm.DbmError):
        ctx.multiply_timing()  # the records were consumed


@pytest.mark.parametrize("bs,side", [(4, 8), (5, 16), (6, 8), (9, 8)])
@pytest.mark.parametrize("kb", [3, 13])
def test_smmq_square_kernel(dbm, ctx, orc, bs, side, kb):
    """The R x R run-square kernel for the padded small sizes (kernels_smmq.cu): a 16R x 16R local grid (256
    squares in Morton order, enough to fill the GPU), kb not a multiple of the stage's k-blocks (the
    zero-predicated tail); integer inputs bit-exact with beta != 0 and beta = 0; U[-1,1) <= 1e-12."""
    n = 16 * side * bs
    for beta in (-1.25, 0.0):
        got, ref, st = run_multiply(dbm, ctx, orc, n, n, kb * bs, bs, "blocked", 0.75, beta, kind=1)
        assert np.array_equal(got, ref)
        assert st["entries"] == (16 * side) ** 2 * kb
    got, ref, _ = run_multiply(dbm, ctx, orc, n, n, kb * bs, bs, "blocked", 0.75, -1.25)
    assert relerr(got, ref) <= TOL
