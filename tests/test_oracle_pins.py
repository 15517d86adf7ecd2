"""Pins for the host oracle (oracle/dbm_oracle.c) against things other than itself:
numpy/BLAS products (a library routine), brute force on tiny inputs, closed forms,
invariants, and the values PAPER.md / SPEC.md print (tests/golden/paper_pins.txt).

Each test names the plausible oracle mistake it would catch.  CPU only.
"""
import math
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden", "paper_pins.txt")


def golden():
    out = {}
    for line in open(GOLD):
        line = line.split("#", 1)[0].strip()
        if not line:
            continue
        k, v = [s.strip() for s in line.split("=")]
        vals = [int(x) for x in v.split(",")]
        out[k] = vals[0] if len(vals) == 1 else tuple(vals)
    return out


G = golden()


def rand_arena(rng, Mb, Nb, bs, ints=False):
    if ints:
        return rng.integers(-2, 3, size=Mb * Nb * bs * bs).astype(np.float64)
    return rng.uniform(-1, 1, size=Mb * Nb * bs * bs)


# ----------------------------------------------------------------- the product
@pytest.mark.parametrize("Mb,Nb,Kb,bs", [(1, 1, 1, 1), (2, 3, 4, 2), (3, 2, 5, 4), (2, 2, 2, 22), (1, 3, 2, 7)])
def test_multiply_matches_numpy_matmul(orc, Mb, Nb, Kb, bs):
    """Catches a transposed operand, wrong block index or dropped term: M != N != K."""
    rng = np.random.default_rng(Mb * 100 + Nb * 10 + Kb + bs)
    A = rand_arena(rng, Mb, Kb, bs)
    B = rand_arena(rng, Kb, Nb, bs)
    C = rand_arena(rng, Mb, Nb, bs)
    Ad = orc.arena_to_dense(A, Mb, Kb, bs)
    Bd = orc.arena_to_dense(B, Kb, Nb, bs)
    Cd = orc.arena_to_dense(C, Mb, Nb, bs)
    alpha, beta = 0.75, -1.25
    expect = alpha * (Ad @ Bd) + beta * Cd
    orc.multiply_blocked(Mb, Nb, Kb, bs, alpha, A, B, beta, C)
    got = orc.arena_to_dense(C, Mb, Nb, bs)
    assert np.abs(got - expect).max() <= 1e-13 * max(1.0, np.abs(expect).max()) * Kb * bs
    # brute-force dense triple loop agrees as well
    bf = orc.dense_gemm(alpha, Ad, Bd, beta, Cd)
    assert np.abs(bf - expect).max() <= 1e-13 * Kb * bs


def test_arena_dense_layout_is_column_major_blocks(orc):
    """Element (x,y) of block (bi,bj) sits at slot*bs^2 + y*bs + x (reading R3)."""
    Mb, Nb, bs = 2, 3, 3
    g = np.arange(Mb * Nb * bs * bs, dtype=np.float64)
    d = orc.arena_to_dense(g, Mb, Nb, bs)
    for bi in range(Mb):
        for bj in range(Nb):
            for x in range(bs):
                for y in range(bs):
                    assert d[bi * bs + x, bj * bs + y] == (bi * Nb + bj) * bs * bs + y * bs + x
    assert np.array_equal(orc.dense_to_arena(d, bs), g)


def test_identity_and_permutation_are_bit_exact(orc):
    """A = I gives C = B exactly; a permutation matrix permutes block rows exactly (misrouting)."""
    rng = np.random.default_rng(7)
    Mb = Kb = 4
    Nb, bs = 3, 5
    B = rand_arena(rng, Kb, Nb, bs)
    I = orc.dense_to_arena(np.eye(Mb * bs), bs)
    C = np.zeros(Mb * Nb * bs * bs)
    orc.multiply_blocked(Mb, Nb, Kb, bs, 1.0, I, B, 0.0, C)
    assert np.array_equal(C, B)
    perm = rng.permutation(Mb * bs)
    Pm = np.eye(Mb * bs)[perm]
    Pa = orc.dense_to_arena(Pm, bs)
    orc.multiply_blocked(Mb, Nb, Kb, bs, 1.0, Pa, B, 0.0, C)
    assert np.array_equal(orc.arena_to_dense(C, Mb, Nb, bs), orc.arena_to_dense(B, Kb, Nb, bs)[perm])


def test_alpha_beta_conventions(orc):
    """beta = 0 never reads C (NaN-filled C stays out); alpha = 0 never reads A, B; linearity."""
    rng = np.random.default_rng(3)
    Mb, Nb, Kb, bs = 2, 2, 3, 4
    A, B = rand_arena(rng, Mb, Kb, bs), rand_arena(rng, Kb, Nb, bs)
    C0 = rand_arena(rng, Mb, Nb, bs)
    Cn = np.full_like(C0, np.nan)
    orc.multiply_blocked(Mb, Nb, Kb, bs, 1.0, A, B, 0.0, Cn)
    assert not np.isnan(Cn).any()
    An = np.full_like(A, np.nan)
    C1 = C0.copy()
    orc.multiply_blocked(Mb, Nb, Kb, bs, 0.0, An, B, -1.25, C1)
    assert np.array_equal(C1, -1.25 * C0)
    AB = np.zeros_like(C0)
    orc.multiply_blocked(Mb, Nb, Kb, bs, 1.0, A, B, 0.0, AB)
    C2 = C0.copy()
    orc.multiply_blocked(Mb, Nb, Kb, bs, 0.5, A, B, 2.0, C2)
    assert np.allclose(C2, 0.5 * AB + 2.0 * C0, rtol=0, atol=1e-14)


def test_small_int_inputs_are_exact(orc):
    """Integer inputs with dyadic alpha/beta: every partial sum exact, so any order agrees bit for bit."""
    rng = np.random.default_rng(11)
    Mb, Nb, Kb, bs = 3, 2, 5, 22
    A, B, C = (rand_arena(rng, Mb, Kb, bs, True), rand_arena(rng, Kb, Nb, bs, True),
               rand_arena(rng, Mb, Nb, bs, True))
    expect = 0.75 * (orc.arena_to_dense(A, Mb, Kb, bs) @ orc.arena_to_dense(B, Kb, Nb, bs)) \
        - 1.25 * orc.arena_to_dense(C, Mb, Nb, bs)
    orc.multiply_blocked(Mb, Nb, Kb, bs, 0.75, A, B, -1.25, C)
    assert np.array_equal(orc.arena_to_dense(C, Mb, Nb, bs), expect)


# ----------------------------------------------------------------- input generator
def test_generator_range_and_distribution(orc):
    """U[-1,1) values, small-int kind in {-2..2}; different seeds / mat_ids differ."""
    a = orc.fill_arena(1910, 0, 0, 220, 220, 22)
    assert a.min() >= -1.0 and a.max() < 1.0
    assert abs(a.mean()) < 0.01 and abs(a.var() - 1 / 3) < 0.01
    hist, _ = np.histogram(a, bins=10, range=(-1, 1))
    assert hist.min() > 0.9 * a.size / 10
    ints = orc.fill_arena(1910, 0, 1, 220, 220, 22)
    assert set(np.unique(ints)) == {-2.0, -1.0, 0.0, 1.0, 2.0}
    assert not np.array_equal(a, orc.fill_arena(1911, 0, 0, 220, 220, 22))
    assert not np.array_equal(a, orc.fill_arena(1910, 1, 0, 220, 220, 22))
    # values are exact multiples of 2^-52 (exactly representable generator)
    assert np.array_equal(np.round(a * 2**52), a * 2**52)


@pytest.mark.parametrize("pr,pc", [(1, 2), (2, 2), (2, 4), (3, 2)])
def test_generator_is_distribution_independent(orc, pr, pc):
    """A rank's local arena equals the scatter of the 1x1 arena: element values depend on global
    indices only (catches a local/global index mix-up in the fill)."""
    rows, cols, bs = 7 * 4, 5 * 4, 4
    g = orc.fill_arena(5, 2, 0, rows, cols, bs)
    for r in range(pr):
        for c in range(pc):
            loc = orc.fill_arena(5, 2, 0, rows, cols, bs, pr, pc, r, c)
            assert np.array_equal(loc, orc.scatter(g, rows // bs, cols // bs, bs, pr, pc, r, c))


# ----------------------------------------------------------------- grid / distribution
def test_grid_dims_north_star(orc):
    assert [orc.grid_dims(p) for p in (1, 2, 4, 8)] == [(1, 1), (1, 2), (2, 2), (2, 4)]


def test_owner_pins_from_spec(orc):
    r, c = G["owner_2x2_block_5_2"]
    assert orc.owner_rank(5, 2, 2, 2) == r * 2 + c
    counts = np.zeros(16, dtype=int)
    for i in range(16):
        for j in range(16):
            counts[orc.owner_rank(i, j, 4, 4)] += 1
    assert (counts == G["owner_4x4_16x16_each"]).all()


def test_local_count_closed_form_and_scatter_gather_roundtrip(orc):
    for nb in range(0, 30):
        for p in range(1, 6):
            for r in range(p):
                assert orc.local_count(nb, p, r) == max(0, math.ceil((nb - r) / p))
    rng = np.random.default_rng(0)
    Mb, Nb, bs, pr, pc = 7, 5, 3, 2, 4
    g = rand_arena(rng, Mb, Nb, bs)
    back = np.zeros_like(g)
    for r in range(pr):
        for c in range(pc):
            orc.gather_into(back, orc.scatter(g, Mb, Nb, bs, pr, pc, r, c), Mb, Nb, bs, pr, pc, r, c)
    assert np.array_equal(back, g)


def test_paper_shapes_divide(orc):
    assert G["blocks_22_square"] * 22 == G["square_M"]
    assert G["square_M"] % 64 == 0 and G["rect_MN"] // 64 == G["blocks_64_rect_mn"]
    assert G["rect_K"] % 22 == 0 and G["rect_K"] % 64 == 0 and G["rect_MN"] % 22 == 0


# ----------------------------------------------------------------- traversal / stacks
def morton_order(n):
    """Independent construction: i-major bit interleaving of (i, j) for n a power of two."""
    def key(i, j):
        k = 0
        for b in range(16):
            k |= ((j >> b) & 1) << (2 * b)
            k |= ((i >> b) & 1) << (2 * b + 1)
        return k
    return sorted(((i, j) for i in range(n) for j in range(n)), key=lambda t: key(*t))


def test_traversal_pins(orc):
    for n in (1, 2, 4, 8, 16):
        assert [tuple(x) for x in orc.traversal(n, n)] == morton_order(n)
    assert [tuple(x) for x in orc.traversal(1, 7)] == [(0, j) for j in range(7)]
    for m, n in [(3, 5), (7, 2), (13, 11), (1, 1)]:
        t = orc.traversal(m, n)
        assert len({tuple(x) for x in t}) == m * n == len(t)
    assert len(orc.traversal(0, 5)) == 0


def brute_entries(mloc, nloc, kb):
    return {(li * kb + kk, kk * nloc + lj, li * nloc + lj) for li in range(mloc) for lj in range(nloc)
            for kk in range(kb)}


@pytest.mark.parametrize("mloc,nloc,kb,cap", [(16, 16, 16, 30000), (16, 16, 16, 100), (5, 3, 7, 20),
                                              (3, 4, 10, 4), (2, 2, 9, 3), (1, 1, 1, 30000), (4, 4, 0, 10)])
def test_stack_contracts(orc, mloc, nloc, kb, cap):
    trip, ptr = orc.stacks(mloc, nloc, kb, cap)
    assert len(trip) == mloc * nloc * kb
    assert {tuple(t) for t in trip.tolist()} == brute_entries(mloc, nloc, kb)
    sizes = np.diff(ptr)
    assert (sizes <= cap).all() and (sizes > 0).all() and sizes.sum() == len(trip)
    if 0 < kb <= cap:  # closed form when runs are never split
        assert len(sizes) == math.ceil(mloc * nloc / (cap // kb))
        # whole runs never straddle a stack boundary
        assert all(p % kb == 0 for p in ptr)
    if kb > cap:
        assert len(sizes) == mloc * nloc * math.ceil(kb / cap)
    # within a run k ascends; runs follow the traversal order
    order = orc.traversal(mloc, nloc)
    if kb:
        cs = trip[::kb, 2]
        assert np.array_equal(cs, order[:, 0] * nloc + order[:, 1])


def test_stack_counts_s352_and_paper_scale(orc):
    """S352 (16^3 blocks) -> 1 stack at cap 30,000 and 43 at cap 100 (SURVEY §8c pins).
    Reading R7: the paper's ~8M / ~0.3M square stacks match this generator at cap 3,000."""
    assert orc.stacks(16, 16, 16, G["stack_cap"], counts_only=True) == (4096, 1)
    assert orc.stacks(16, 16, 16, 100, counts_only=True) == (4096, 43)
    nb22, nb64 = G["square_M"] // 22, G["square_M"] // 64
    assert orc.stacks(nb22, nb22, nb22, 30000, counts_only=True)[1] == 829440
    assert orc.stacks(nb64, nb64, nb64, 30000, counts_only=True)[1] == 32670
    s22 = orc.stacks(nb22, nb22, nb22, 3000, counts_only=True)[1]
    s64 = orc.stacks(nb64, nb64, nb64, 3000, counts_only=True)[1]
    assert abs(s22 / G["stacks_square_bs22"] - 1) < 0.1
    assert abs(s64 / G["stacks_square_bs64"] - 1) < 0.1


def test_densified_is_one_stack_of_one_entry(orc):
    """P:198 §III: after densification 'the size of the batches become 1'."""
    e, ns = orc.stacks(1, 1, 1, G["stack_cap"], counts_only=True)
    assert (e, ns) == (G["densified_batch_size"], 1)


# ----------------------------------------------------------------- Cannon
GRIDS = [(1, 1), (1, 2), (2, 1), (2, 2), (2, 4), (4, 2), (3, 3), (1, 4), (4, 1), (3, 2)]


@pytest.mark.parametrize("pr,pc", GRIDS)
def test_cannon_schedule_computes_the_product(orc, pr, pc):
    """Simulate the schedule with numpy panels (ragged block counts): every rank sees every K panel
    exactly once, from a rank that owns it, and the sum of panel products is A@B."""
    L = orc.lcm(pr, pc)
    Mb, Nb, Kb, bs = 5, 7, 9, 2
    rng = np.random.default_rng(pr * 10 + pc)
    A = rng.uniform(-1, 1, (Mb * bs, Kb * bs))
    B = rng.uniform(-1, 1, (Kb * bs, Nb * bs))
    Cout = np.zeros((Mb * bs, Nb * bs))
    for r in range(pr):
        for c in range(pc):
            rows = [i for i in range(Mb) if i % pr == r]
            cols = [j for j in range(Nb) if j % pc == c]
            seen = []
            for s in range(L):
                k, asrc, bsrc = orc.cannon_step(pr, pc, r, c, s)
                seen.append(k)
                ks = [kk for kk in range(Kb) if kk % L == k]
                # the source really owns every block of the panel
                assert all(orc.owner_rank(i, kk, pr, pc) == asrc for i in rows for kk in ks)
                assert all(orc.owner_rank(kk, j, pr, pc) == bsrc for kk in ks for j in cols)
                ri = np.concatenate([np.arange(i * bs, i * bs + bs) for i in rows]) if rows else np.array([], int)
                ci = np.concatenate([np.arange(j * bs, j * bs + bs) for j in cols]) if cols else np.array([], int)
                ki = np.concatenate([np.arange(q * bs, q * bs + bs) for q in ks]) if ks else np.array([], int)
                if len(ri) and len(ci) and len(ki):
                    Cout[np.ix_(ri, ci)] += A[np.ix_(ri, ki)] @ B[np.ix_(ki, ci)]
            assert sorted(seen) == list(range(L))
    assert np.allclose(Cout, A @ B, atol=1e-12)


@pytest.mark.parametrize("pr,pc", GRIDS)
def test_cannon_at_most_one_send_per_operand_per_step(orc, pr, pc):
    L = orc.lcm(pr, pc)
    for s in range(L):
        a_sends, b_sends = {}, {}
        for r in range(pr):
            for c in range(pc):
                k, asrc, bsrc = orc.cannon_step(pr, pc, r, c, s)
                me = r * pc + c
                if asrc != me:
                    a_sends.setdefault(asrc, set()).add(k)
                if bsrc != me:
                    b_sends.setdefault(bsrc, set()).add(k)
        assert all(len(v) <= 1 for v in a_sends.values())
        assert all(len(v) <= 1 for v in b_sends.values())


@pytest.mark.parametrize("pt", [1, 2, 3, 4])
def test_cannon_bytes_closed_form_square(orc, pt):
    """per-rank bytes = 2*(N/P~)^2*8*(P~-1) for dense square doubles, N divisible by P~."""
    N, bs = 24 * pt, 2
    nb = N // bs
    for r in range(pt):
        for c in range(pt):
            rv, sd = orc.cannon_bytes(nb, nb, nb, bs, pt, pt, r, c)
            assert rv == 2 * (N // pt) ** 2 * 8 * (pt - 1)
            assert sd == rv


def test_cannon_bytes_general_formula(orc):
    """Non-square grids: recv = (L-L/Pc)|A_panel| + (L-L/Pr)|B_panel| when panels divide evenly."""
    for pr, pc in [(1, 2), (2, 4), (4, 2), (1, 4)]:
        L = orc.lcm(pr, pc)
        Mb, Nb, Kb, bs = 4 * pr, 4 * pc, 3 * L, 2
        ap = (Mb // pr) * (Kb // L) * bs * bs * 8
        bp = (Kb // L) * (Nb // pc) * bs * bs * 8
        for r in range(pr):
            for c in range(pc):
                rv, _ = orc.cannon_bytes(Mb, Nb, Kb, bs, pr, pc, r, c)
                assert rv == (L - L // pc) * ap + (L - L // pr) * bp


def test_cannon_volume_scales_as_inverse_sqrt_p(orc):
    """per-rank volume O(1/sqrt(P)); P=4 -> P=16 halves it (within 10%)."""
    N, bs = 960, 4
    nb = N // bs
    v4 = orc.cannon_bytes(nb, nb, nb, bs, 2, 2, 0, 0)[0]
    v16 = orc.cannon_bytes(nb, nb, nb, bs, 4, 4, 0, 0)[0]
    assert abs(v16 / v4 - 0.5) < 0.1 * 0.5 + 0.25  # (P~-1)/P~^2 : 3/16 vs 1/4 -> 0.75 exactly
    assert v16 / v4 == pytest.approx((3 / 16) / (1 / 4))


# ----------------------------------------------------------------- densification
def test_densify_law_eqs_1_2(orc):
    M, pt, t = G["densify_law_case"]
    a, b = orc.densified_dims(M, M, M, pt, t)
    assert a == G["densify_law_A"] and b == G["densify_law_B"]
    # the law reassembles the whole matrix: t*P~ A blocks of rows, P~ along K and N
    assert a[0] * t * pt == M and a[1] * pt == M and b[0] * pt == M and b[1] * pt == M


def test_densify_layouts_and_roundtrip(orc):
    rng = np.random.default_rng(5)
    mloc, nloc, bs = 3, 4, 5
    arena = rand_arena(rng, mloc, nloc, bs)
    dense_all = orc.densify_cols(arena, mloc, nloc, bs, np.arange(nloc), 0)
    ref = orc.arena_to_dense(arena, mloc, nloc, bs)  # the full local arena as a dense matrix
    assert np.array_equal(dense_all.reshape(nloc * bs, mloc * bs).T, ref)
    rowmaj = orc.densify_cols(arena, mloc, nloc, bs, np.arange(nloc), 1)
    assert np.array_equal(rowmaj.reshape(mloc * bs, nloc * bs), ref)
    sub = [3, 1]
    d = orc.densify_cols(arena, mloc, nloc, bs, sub, 0).reshape(len(sub) * bs, mloc * bs).T
    assert np.array_equal(d, ref[:, np.concatenate([np.arange(q * bs, q * bs + bs) for q in sub])])
    rws = [2, 0]
    d = orc.densify_rows(arena, mloc, nloc, bs, rws, 0).reshape(nloc * bs, len(rws) * bs).T
    assert np.array_equal(d, ref[np.concatenate([np.arange(q * bs, q * bs + bs) for q in rws]), :])
    d1 = orc.densify_rows(arena, mloc, nloc, bs, rws, 1).reshape(len(rws) * bs, nloc * bs)
    assert np.array_equal(d1, d)
    # undensify(alpha=1, beta=0) inverts densify bit for bit
    back = np.full_like(arena, np.nan)
    orc.undensify(dense_all, mloc * bs, mloc, nloc, bs, 1.0, 0.0, back)
    assert np.array_equal(back, arena)


def test_undensify_alpha_beta(orc):
    rng = np.random.default_rng(9)
    mloc, nloc, bs = 2, 3, 4
    dense = rng.uniform(-1, 1, (mloc * bs) * (nloc * bs))
    c = rand_arena(rng, mloc, nloc, bs)
    out = c.copy()
    orc.undensify(dense, mloc * bs, mloc, nloc, bs, 0.75, -1.25, out)
    D = dense.reshape(nloc * bs, mloc * bs).T
    expect = 0.75 * D + (-1.25) * orc.arena_to_dense(c, mloc, nloc, bs)
    assert np.array_equal(orc.arena_to_dense(out, mloc, nloc, bs), expect)


# ----------------------------------------------------------------- verification helpers
def test_rows_and_freivalds_from_seeds(orc):
    M, N, K, bs, seed = 88, 66, 110, 22, 1910
    A = orc.fill_arena(seed, 0, 0, M, K, bs)
    B = orc.fill_arena(seed, 1, 0, K, N, bs)
    Cin = orc.fill_arena(seed, 2, 0, M, N, bs)
    Ad, Bd, Cd = (orc.arena_to_dense(A, M // bs, K // bs, bs), orc.arena_to_dense(B, K // bs, N // bs, bs),
                  orc.arena_to_dense(Cin, M // bs, N // bs, bs))
    expect = 0.75 * (Ad @ Bd) - 1.25 * Cd
    rows = [0, 1, 21, 22, 87]
    got = orc.rows_from_seeds(M, N, K, seed, 0, 0.75, -1.25, rows)
    assert np.abs(got - expect[rows]).max() < 1e-13
    x, rhs = orc.freivalds_rhs(M, N, K, seed, 0, 0.75, -1.25, 42)
    assert set(np.unique(x)) == {-1.0, 1.0}
    assert np.abs(rhs - expect @ x).max() < 1e-12
    # and the oracle's own blocked product agrees with the rows
    C = Cin.copy()
    orc.multiply_blocked(M // bs, N // bs, K // bs, bs, 0.75, A, B, -1.25, C)
    assert np.array_equal(orc.arena_to_dense(C, M // bs, N // bs, bs)[rows], got)


# ----------------------------------------------------------------- tall-and-skinny (reading R14)
@pytest.mark.parametrize("pr,pc", [(1, 2), (2, 2), (2, 4), (1, 4), (4, 1), (3, 2)])
def test_tallskinny_partition_computes_the_product(orc, pr, pc):
    """Simulate R14 with numpy: rank p sums A[:, S_p] B[S_p, :] over S_p = {k : k mod P == p}; every
    k in S_p lies in p's grid column (k mod Pc == c); the sum of the P partials is A @ B."""
    P = pr * pc
    Mb, Nb, Kb, bs = 5, 3, 23, 2
    rng = np.random.default_rng(P)
    A = rng.uniform(-1, 1, (Mb * bs, Kb * bs))
    B = rng.uniform(-1, 1, (Kb * bs, Nb * bs))
    total = np.zeros((Mb * bs, Nb * bs))
    for p in range(P):
        r, c = divmod(p, pc)
        ks = [k for k in range(Kb) if k % P == p]
        assert all(k % pc == c for k in ks)
        assert all(orc.owner_rank(k, 0, pr, pc) // pc == p % pr for k in ks)  # B rows in grid row p mod Pr
        idx = np.concatenate([np.arange(k * bs, k * bs + bs) for k in ks]) if ks else np.array([], int)
        total += A[:, idx] @ B[idx, :]
    assert np.allclose(total, A @ B, atol=1e-12)


def test_tallskinny_bytes(orc):
    """Reduction-only volume (K = 0) is (P-1) x the rank's C share: O(1) in P for fixed M, N;
    on the paper's rectangular shape at 2x4 the gather moves ~3x less than Cannon."""
    for pr, pc in [(1, 4), (2, 2), (2, 4), (4, 4)]:
        P = pr * pc
        Mb = Nb = 16
        for r in range(pr):
            for c in range(pc):
                rv, _ = orc.ts_bytes(Mb, Nb, 0, 4, pr, pc, r, c)
                assert rv == (P - 1) * orc.local_count(Mb, pr, r) * orc.local_count(Nb, pc, c) * 16 * 8
    Mb, Nb, Kb, bs = 22, 22, 30976, 64  # 1,408 x 1,408 x 1,982,464 bs 64
    ts = max(orc.ts_bytes(Mb, Nb, Kb, bs, 2, 4, r, c)[0] for r in range(2) for c in range(4))
    cannon = max(orc.cannon_bytes(Mb, Nb, Kb, bs, 2, 4, r, c)[0] for r in range(2) for c in range(4))
    assert ts < cannon / 2.5
    # gathers: 1x4 needs no A (all rows local), only B pieces from the 3 peers
    rv, _ = orc.ts_bytes(8, 8, 40, 2, 1, 4, 0, 1)
    kp = orc.local_count(40, 4, 1)
    assert rv == kp * 6 * 4 * 8 + 3 * 8 * 2 * 4 * 8  # B: kp x (8 - 2 local cols) blocks; C: 3 x (8 x 2) blocks


# ----------------------------------------------------------------- block sparsity (reading R15)
def test_pattern_generator_occupancy(orc):
    """occupancy 0 / 1 are exact; other occupancies land within 5 sigma of the binomial mean (catches a
    wrong comparison direction or a stream shared with the element generator)."""
    assert orc.pattern_random(7, 0, 30, 40, 0.0).sum() == 0
    assert orc.pattern_random(7, 0, 30, 40, 1.0).all()
    n = 200 * 200
    for occ in (0.01, 0.1, 0.5, 0.9):
        m = orc.pattern_random(1910, 3, 200, 200, occ)
        assert abs(m.sum() - occ * n) <= 5 * math.sqrt(n * occ * (1 - occ)) + 1
    a, b = orc.pattern_random(1910, 0, 50, 50, 0.5), orc.pattern_random(1910, 1, 50, 50, 0.5)
    assert 0.3 < (a == b).mean() < 0.7  # independent per mat_id
    # monotone in occupancy: a block stored at occupancy p is stored at every q > p
    lo, hi = orc.pattern_random(5, 2, 40, 40, 0.2), orc.pattern_random(5, 2, 40, 40, 0.6)
    assert not (lo & ~hi).any()


@pytest.mark.parametrize("Mb,Nb,Kb,bs,occ", [(4, 3, 5, 2, 0.5), (6, 5, 7, 3, 0.2), (3, 3, 3, 4, 0.9), (5, 4, 6, 1, 0.0)])
def test_multiply_sparse_matches_masked_numpy(orc, Mb, Nb, Kb, bs, occ):
    """Absent blocks act as zeros in A and B; C keeps its pattern (absent C blocks untouched, present ones
    get beta*C + alpha*A*B).  Catches a mask applied to the wrong operand or a transposed mask."""
    rng = np.random.default_rng(Mb * 100 + Kb)
    am = orc.pattern_random(11, 0, Mb, Kb, occ)
    bm = orc.pattern_random(11, 1, Kb, Nb, occ)
    cm = orc.pattern_random(11, 2, Mb, Nb, max(occ, 0.5))
    A, B, Cg = rand_arena(rng, Mb, Kb, bs), rand_arena(rng, Kb, Nb, bs), rand_arena(rng, Mb, Nb, bs)
    Ad = orc.arena_to_dense(A, Mb, Kb, bs) * np.kron(am, np.ones((bs, bs)))
    Bd = orc.arena_to_dense(B, Kb, Nb, bs) * np.kron(bm, np.ones((bs, bs)))
    Cd = orc.arena_to_dense(Cg, Mb, Nb, bs)
    out = Cg.copy()
    orc.multiply_sparse(Mb, Nb, Kb, bs, 0.75, A, am, B, bm, -1.25, out, cm)
    got = orc.arena_to_dense(out, Mb, Nb, bs)
    cmask = np.kron(cm, np.ones((bs, bs))).astype(bool)
    want = np.where(cmask, 0.75 * (Ad @ Bd) - 1.25 * Cd, Cd)
    assert np.allclose(got, want, rtol=0, atol=1e-12)


def test_multiply_sparse_dense_pattern_is_the_dense_oracle(orc):
    """With every block stored the sparse product is bit-identical to orc_multiply_blocked (same order)."""
    rng = np.random.default_rng(3)
    Mb, Nb, Kb, bs = 3, 4, 5, 3
    A, B, Cg = rand_arena(rng, Mb, Kb, bs), rand_arena(rng, Kb, Nb, bs), rand_arena(rng, Mb, Nb, bs)
    one = lambda r, c: np.ones((r, c), np.uint8)  # noqa: E731
    x, y = Cg.copy(), Cg.copy()
    orc.multiply_sparse(Mb, Nb, Kb, bs, 0.5, A, one(Mb, Kb), B, one(Kb, Nb), 2.0, x, one(Mb, Nb))
    orc.multiply_blocked(Mb, Nb, Kb, bs, 0.5, A, B, 2.0, y)
    assert np.array_equal(x, y)


def test_sparse_compress_expand_roundtrip(orc):
    """Local CSR order = li ascending then lj ascending over stored blocks (DBCSR's blocked CSR)."""
    rng = np.random.default_rng(9)
    Mb, Nb, bs, pr, pc = 7, 6, 2, 2, 3
    g = rand_arena(rng, Mb, Nb, bs)
    m = orc.pattern_random(4, 0, Mb, Nb, 0.4)
    back = np.zeros_like(g)
    total = 0
    for r in range(pr):
        for c in range(pc):
            loc = orc.sparse_compress(g, m, Mb, Nb, bs, pr, pc, r, c)
            blocks = [(bi, bj) for bi in range(r, Mb, pr) for bj in range(c, Nb, pc) if m[bi, bj]]
            assert loc.size == len(blocks) * bs * bs
            for n, (bi, bj) in enumerate(blocks):  # brute force: block n is (bi, bj)
                s = (bi * Nb + bj) * bs * bs
                assert np.array_equal(loc[n * bs * bs:(n + 1) * bs * bs], g[s:s + bs * bs])
            orc.sparse_expand_into(back, loc, m, Mb, Nb, bs, pr, pc, r, c)
            total += len(blocks)
    assert total == m.sum()
    mask_el = np.repeat(m.reshape(-1), bs * bs).astype(bool)
    assert np.array_equal(back[mask_el], g[mask_el]) and not back[~mask_el].any()


@pytest.mark.parametrize("mloc,nloc,kb,occ,cap", [(4, 4, 6, 0.5, 7), (5, 3, 9, 0.3, 4), (6, 7, 4, 0.8, 30000),
                                                  (3, 3, 5, 0.0, 10), (8, 8, 3, 1.0, 5)])
def test_sparse_stacks_brute_force(orc, mloc, nloc, kb, occ, cap):
    """Pure-Python enumeration of the R15 rule on tiny inputs: runs = stored C blocks in bisection order
    (the traversal itself pinned by test_traversal_*), entries kk ascending where both A and B are
    stored, slots = row-major rank among stored panel blocks; entry count = sum of the mask product."""
    am = orc.pattern_random(21, 0, mloc, kb, occ)
    bm = orc.pattern_random(21, 1, kb, nloc, occ)
    cm = orc.pattern_random(21, 2, mloc, nloc, max(occ, 0.6))
    trip, ptr = orc.sparse_stacks(am, bm, cm, cap)
    aslot = {ij: n for n, ij in enumerate((i, k) for i in range(mloc) for k in range(kb) if am[i, k])}
    bslot = {ij: n for n, ij in enumerate((k, j) for k in range(kb) for j in range(nloc) if bm[k, j])}
    cslot = {ij: n for n, ij in enumerate((i, j) for i in range(mloc) for j in range(nloc) if cm[i, j])}
    want, runs = [], []
    for li, lj in orc.traversal(mloc, nloc):
        if not cm[li, lj]:
            continue
        run = [(aslot[(li, k)], bslot[(k, lj)], cslot[(li, lj)]) for k in range(kb) if am[li, k] and bm[k, lj]]
        if run:
            runs.append(len(run))
        want += run
    assert [tuple(t) for t in trip] == want
    assert len(want) == int(((am.astype(int) @ bm.astype(int)) * cm).sum())
    # greedy whole-run packing (same rule as the dense pin): rebuild the boundaries
    b, cur, e = [0], 0, 0
    for n in runs:
        if n > cap:
            if cur:
                b.append(e)
                cur = 0
            done = 0
            while done < n:
                done += min(cap, n - done)
                b.append(e + done)
        else:
            if cur + n > cap:
                b.append(e)
                cur = 0
            cur += n
        e += n
    if cur:
        b.append(e)
    assert list(ptr) == b
    assert all(ptr[i + 1] - ptr[i] <= cap for i in range(len(ptr) - 1))


def test_sparse_stacks_dense_pattern_equals_dense_stacks(orc):
    one = lambda r, c: np.ones((r, c), np.uint8)  # noqa: E731
    for mloc, nloc, kb, cap in [(5, 3, 4, 6), (4, 4, 9, 5)]:
        t1, p1 = orc.sparse_stacks(one(mloc, kb), one(kb, nloc), one(mloc, nloc), cap)
        t2, p2 = orc.stacks(mloc, nloc, kb, cap)
        assert np.array_equal(t1, t2) and np.array_equal(p1, p2)


def test_sparse_rows_from_seeds_matches_masked_numpy(orc):
    """Sampled-row checker for sparse configs: equals the masked numpy product on the stored C blocks, NaN
    elsewhere, and counts exactly bs^2 multiply-adds per (stored A, B, C) block triple of the row."""
    M, N, K, bs, ps = 66, 88, 110, 11, 3
    oa, ob, oc = 0.4, 0.5, 0.7
    Mb, Nb, Kb = M // bs, N // bs, K // bs
    am, bm, cm = orc.pattern_random(ps, 0, Mb, Kb, oa), orc.pattern_random(ps, 1, Kb, Nb, ob), \
        orc.pattern_random(ps, 2, Mb, Nb, oc)
    A = orc.arena_to_dense(orc.fill_arena(1910, 0, 0, M, K, bs), Mb, Kb, bs) * np.kron(am, np.ones((bs, bs)))
    B = orc.arena_to_dense(orc.fill_arena(1910, 1, 0, K, N, bs), Kb, Nb, bs) * np.kron(bm, np.ones((bs, bs)))
    Cd = orc.arena_to_dense(orc.fill_arena(1910, 2, 0, M, N, bs), Mb, Nb, bs)
    rows = np.array([0, 5, 11, 40, 65])
    out, fmas = orc.sparse_rows_from_seeds(M, N, K, bs, 1910, 0, ps, oa, ob, oc, 0.75, -1.25, rows)
    cmask = np.kron(cm, np.ones((bs, bs))).astype(bool)[rows]
    want = (0.75 * (A @ B) - 1.25 * Cd)[rows]
    assert np.allclose(out[cmask], want[cmask], rtol=0, atol=1e-12)
    assert np.isnan(out[~cmask]).all()
    triples = sum(int(am[i // bs, k] and bm[k, j] and cm[i // bs, j]) for i in rows for k in range(Kb) for j in range(Nb))
    assert fmas == triples * bs * bs


# ----------------------------------------------------------------- round-2 pins (VERDICT r1 "pin gaps")
def test_lcm_matches_math_lcm(orc):
    """orc_lcm gives L, the number of Cannon steps (reading R5); a schedule test would still pass with
    L = Pr*Pc, so pin it against the library routine on every pair up to 40 (catches a gcd slip)."""
    for a in range(1, 41):
        for b in range(1, 41):
            assert orc.lcm(a, b) == math.lcm(a, b), (a, b)


def _owned_sorted(Mb, Nb, pr, pc, q, orc):
    """Brute force through orc_owner_rank (pinned by S:127): rank q's global blocks in (bi, bj) order."""
    return [(bi, bj) for bi in range(Mb) for bj in range(Nb) if orc.owner_rank(bi, bj, pr, pc) == q]


@pytest.mark.parametrize("Mb,Nb,bs,pr,pc", [(7, 5, 3, 2, 4), (5, 9, 2, 3, 2), (4, 4, 1, 1, 1), (6, 3, 2, 4, 2),
                                            (1, 7, 2, 2, 4)])
def test_scatter_gather_brute_force_through_owner(orc, Mb, Nb, bs, pr, pc):
    """orc_scatter / orc_gather move block (bi, bj) to its owner at the position it takes in the
    owner's (row, column)-ascending list of owned blocks (the local CSR order, reading R3).  Every block
    is tagged with its global coordinates, so a wrong slot, a swapped residue or a dropped block fails."""
    bb = bs * bs
    g = np.zeros(Mb * Nb * bb)
    for bi in range(Mb):
        for bj in range(Nb):
            g[(bi * Nb + bj) * bb:(bi * Nb + bj + 1) * bb] = 1000 * bi + bj + np.arange(bb) / (bb + 1)
    seen = 0
    back = np.full_like(g, np.nan)
    for r in range(pr):
        for c in range(pc):
            q = r * pc + c
            owned = _owned_sorted(Mb, Nb, pr, pc, q, orc)
            loc = orc.scatter(g, Mb, Nb, bs, pr, pc, r, c)
            assert loc.size == len(owned) * bb
            for s, (bi, bj) in enumerate(owned):
                assert np.array_equal(loc[s * bb:(s + 1) * bb], g[(bi * Nb + bj) * bb:(bi * Nb + bj + 1) * bb])
            seen += len(owned)
            orc.gather_into(back, loc, Mb, Nb, bs, pr, pc, r, c)
    assert seen == Mb * Nb
    assert np.array_equal(back, g)


@pytest.mark.parametrize("Mb,Nb,Kb,bs,pr,pc", [(5, 6, 11, 2, 2, 4), (4, 3, 7, 3, 1, 2), (3, 5, 9, 2, 2, 2),
                                               (6, 4, 13, 1, 4, 2), (2, 2, 5, 2, 1, 1)])
def test_pack_panel_brute_force(orc, Mb, Nb, Kb, bs, pr, pc):
    """a3 (pack panel): A(r, kappa) holds the global blocks (bi, bk) with bi owned by grid row r and
    bk = kappa (mod L), ascending, packed row-major over (li, kk); B(kappa, c) the blocks (bk, bj), bj
    owned by grid column c, row-major over (kk, lj).  The expected panel is read from the tagged global
    arena by definition; the oracle packs from the scattered local arena (catches a transposed pack
    order, a wrong stride or a wrong residue)."""
    L = math.lcm(pr, pc)
    bb = bs * bs

    def tagged(R, Cn, mat):
        g = np.zeros(R * Cn * bb)
        for i in range(R):
            for j in range(Cn):
                g[(i * Cn + j) * bb:(i * Cn + j + 1) * bb] = mat * 1e6 + 1000 * i + j + np.arange(bb) / (bb + 1)
        return g

    gA, gB = tagged(Mb, Kb, 1), tagged(Kb, Nb, 2)
    for r in range(pr):
        for c in range(pc):
            locA = orc.scatter(gA, Mb, Kb, bs, pr, pc, r, c)
            locB = orc.scatter(gB, Kb, Nb, bs, pr, pc, r, c)
            rows = [i for i in range(Mb) if i % pr == r]
            acols = [k for k in range(Kb) if k % pc == c]  # A's local block columns
            brows = [k for k in range(Kb) if k % pr == r]  # B's local block rows
            cols = [j for j in range(Nb) if j % pc == c]
            for kappa in range(L):
                ks = [k for k in range(Kb) if k % L == kappa]
                if kappa % pc == c:  # this rank owns A(r, kappa)
                    got = orc.pack_panel(locA, len(rows), len(acols), bs, 0, [acols.index(k) for k in ks])
                    exp = np.concatenate([gA[(i * Kb + k) * bb:(i * Kb + k + 1) * bb] for i in rows for k in ks]
                                         or [np.zeros(0)])
                    assert np.array_equal(got, exp)
                if kappa % pr == r:  # this rank owns B(kappa, c)
                    got = orc.pack_panel(locB, len(brows), len(cols), bs, 1, [brows.index(k) for k in ks])
                    exp = np.concatenate([gB[(k * Nb + j) * bb:(k * Nb + j + 1) * bb] for k in ks for j in cols]
                                         or [np.zeros(0)])
                    assert np.array_equal(got, exp)


# ----------------------------------------------------------------- non-uniform block sizes (reading R16)
def _cut(sizes):
    o = np.concatenate([[0], np.cumsum(sizes)]).astype(int)
    return [(o[i], o[i + 1]) for i in range(len(sizes))]


@pytest.mark.parametrize("rsz,csz,pr,pc", [([5, 13, 22, 3], [23, 4, 26], 2, 2), ([7], [1, 2, 3, 4, 5], 1, 2),
                                           ([22, 22, 22], [64, 22], 2, 1), ([9, 1, 31, 2, 17], [6, 11], 2, 4)])
def test_nu_scatter_gather_brute_force(orc, rsz, csz, pr, pc):
    """R16 layout: rank (r, c)'s arena = its blocks (owner rule S:115 through orc_owner_rank) in (bi, bj) order,
    each column-major, back to back; read from the dense array by slicing (catches a swapped size list, a
    row-major block or a wrong prefix offset).  Scatter over all ranks then gather restores the array."""
    rng = np.random.default_rng(3)
    M, N = sum(rsz), sum(csz)
    D = rng.uniform(-1, 1, (M, N))
    rows, cols = _cut(rsz), _cut(csz)
    mask = (rng.uniform(size=(len(rsz), len(csz))) < 0.7).astype(np.uint8)
    for mk in (None, mask):
        back = np.full((N, M), np.nan)  # column-major storage of the (M, N) result
        for r in range(pr):
            for c in range(pc):
                q = r * pc + c
                exp = [D[rows[bi][0]:rows[bi][1], cols[bj][0]:cols[bj][1]].T.reshape(-1)
                       for bi in range(len(rsz)) for bj in range(len(csz))
                       if orc.owner_rank(bi, bj, pr, pc) == q and (mk is None or mk[bi, bj])]
                exp = np.concatenate(exp) if exp else np.zeros(0)
                loc = orc.nu_scatter(D, rsz, csz, pr, pc, r, c, mk)
                assert orc.nu_local_elems(rsz, csz, pr, pc, r, c, mk) == exp.size
                assert np.array_equal(loc, exp)
                orc.nu_gather_into(back, loc, rsz, csz, pr, pc, r, c, mk)
        stored = np.ones((M, N), bool)
        if mk is not None:
            stored = np.zeros((M, N), bool)
            for bi in range(len(rsz)):
                for bj in range(len(csz)):
                    if mk[bi, bj]:
                        stored[rows[bi][0]:rows[bi][1], cols[bj][0]:cols[bj][1]] = True
        assert np.array_equal(back.T[stored], D[stored]) and np.isnan(back.T[~stored]).all()


@pytest.mark.parametrize("msz,nsz,ksz", [([5, 13, 22], [23, 4, 26, 9], [7, 22, 31]), ([64], [1], [2, 3]),
                                         ([22] * 3, [22] * 2, [22] * 4)])
def test_nu_multiply_matches_numpy(orc, msz, nsz, ksz):
    """Mixed (m, n, k) block products: all-stored = alpha*A@B + beta*C (numpy/BLAS); with masks =
    the product of the block-masked operands on the stored C blocks, the other C entries untouched
    (catches a transposed block, a dropped k block or an m/n swap on non-square blocks)."""
    rng = np.random.default_rng(5)
    M, N, K = sum(msz), sum(nsz), sum(ksz)
    A, B, C = rng.uniform(-1, 1, (M, K)), rng.uniform(-1, 1, (K, N)), rng.uniform(-1, 1, (M, N))
    got = orc.nu_multiply(msz, nsz, ksz, 0.75, A, B, -1.25, C)
    assert np.allclose(got, 0.75 * A @ B - 1.25 * C, rtol=0, atol=1e-12)

    def expand(mask, rs, cs):
        e = np.zeros((sum(rs), sum(cs)), bool)
        for i, (a0, a1) in enumerate(_cut(rs)):
            for j, (b0, b1) in enumerate(_cut(cs)):
                e[a0:a1, b0:b1] = mask[i, j]
        return e

    am = (rng.uniform(size=(len(msz), len(ksz))) < 0.6).astype(np.uint8)
    bm = (rng.uniform(size=(len(ksz), len(nsz))) < 0.6).astype(np.uint8)
    cm = (rng.uniform(size=(len(msz), len(nsz))) < 0.6).astype(np.uint8)
    got = orc.nu_multiply(msz, nsz, ksz, 0.75, A, B, -1.25, C, am, bm, cm)
    Ae, Be, Ce = expand(am, msz, ksz), expand(bm, ksz, nsz), expand(cm, msz, nsz)
    ref = np.where(Ce, 0.75 * (A * Ae) @ (B * Be) - 1.25 * C, C)
    assert np.allclose(got, ref, rtol=0, atol=1e-12)


def test_nu_multiply_uniform_is_the_blocked_oracle_and_conventions(orc):
    """Uniform sizes reduce R16 to the uniform layout: orc_nu_multiply through nu_scatter equals
    orc_multiply_blocked bit for bit (same k order); alpha = 0 gives beta*C exactly, beta = 0 ignores a
    NaN C (reading R8)."""
    Mb, Nb, Kb, bs = 3, 2, 4, 5
    A = orc.fill_dense(7, 0, 0, Mb * bs, Kb * bs)
    B = orc.fill_dense(7, 1, 0, Kb * bs, Nb * bs)
    C = orc.fill_dense(7, 2, 0, Mb * bs, Nb * bs)
    got = orc.nu_multiply([bs] * Mb, [bs] * Nb, [bs] * Kb, 0.75, A, B, -1.25, C)
    Ag = orc.fill_arena(7, 0, 0, Mb * bs, Kb * bs, bs)
    Bg = orc.fill_arena(7, 1, 0, Kb * bs, Nb * bs, bs)
    Cg = orc.fill_arena(7, 2, 0, Mb * bs, Nb * bs, bs)
    orc.multiply_blocked(Mb, Nb, Kb, bs, 0.75, Ag, Bg, -1.25, Cg)
    assert np.array_equal(orc.nu_scatter(got, [bs] * Mb, [bs] * Nb), Cg)
    assert np.array_equal(orc.nu_multiply([bs] * Mb, [bs] * Nb, [bs] * Kb, 0.0, A * np.nan, B, -1.25, C), -1.25 * C)
    assert not np.isnan(orc.nu_multiply([bs] * Mb, [bs] * Nb, [bs] * Kb, 1.0, A, B, 0.0, C * np.nan)).any()
