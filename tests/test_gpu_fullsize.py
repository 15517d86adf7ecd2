"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times (one GPU):
the oracle recomputes sampled rows of C from the seeds (rows at 0, M-1, block edges and spread
through the matrix) and a Freivalds check compares C_out x with alpha*A(Bx) + beta*C_in x for a
seeded +-1 vector x.  Tolerance 1e-12 normwise relative (north star); with the small-integer inputs
both checks are exact.  The GPU-side matrix-vector product is test-side torch (einsum on the
output arena); the expected values come only from oracle/.
"""
import numpy as np
import pytest
import torch

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

SEED = 1910
TOL = 1e-12


@pytest.fixture(scope="module")
def dbm():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1910_04796_b200 as d

    d.load()
    return d


def sample_rows(M, bs, n=12):
    rows = {0, M - 1, bs - 1, bs, M // 2, M // 2 + 1, M - bs}
    rng = np.random.default_rng(7)
    rows |= set(rng.integers(0, M, n).tolist())
    return np.array(sorted(rows), dtype=np.int64)


def gpu_rows(C, rows, bs):
    """Rows of the dense C from the 1x1 arena: C[bi*bs+x, bj*bs+y] = arena[bi, bj, y, x]."""
    Mb, Nb = C.rows // bs, C.cols // bs
    a = C.arena[: Mb * Nb * bs * bs].view(Mb, Nb, bs, bs)
    r = torch.as_tensor(rows, device=a.device)
    blk = a[r // bs, :, :, r % bs]  # (nrows, Nb, bs(y))
    return blk.reshape(len(rows), Nb * bs).cpu().numpy()


def gpu_matvec(C, x, bs):
    Mb, Nb = C.rows // bs, C.cols // bs
    a = C.arena[: Mb * Nb * bs * bs].view(Mb, Nb, bs, bs)
    xv = torch.as_tensor(x, device=a.device).view(Nb, bs)
    return torch.einsum("ijyx,jy->ix", a, xv).reshape(-1).cpu().numpy()


def run_and_check(dbm, orc, M, N, K, bs, path, kind, alpha=0.75, beta=-1.25):
    ctx = dbm.Context()
    A, B, C = dbm.Matrix(ctx, M, K, bs), dbm.Matrix(ctx, K, N, bs), dbm.Matrix(ctx, M, N, bs)
    A.fill_random(SEED, 0, kind)
    B.fill_random(SEED, 1, kind)
    C.fill_random(SEED, 2, kind)
    x_seed = 4242
    x, rhs = orc.freivalds_rhs(M, N, K, SEED, kind, alpha, beta, x_seed)  # uses C_in from its seed
    rows = sample_rows(M, bs)
    ref_rows = orc.rows_from_seeds(M, N, K, SEED, kind, alpha, beta, rows)
    dbm.multiply(ctx, alpha, A, B, beta, C, path)
    ctx.sync()
    got_rows = gpu_rows(C, rows, bs)
    lhs = gpu_matvec(C, x, bs)
    ctx.release_workspace()
    del A, B
    if kind == 1:
        assert np.array_equal(got_rows, ref_rows)
        assert np.array_equal(lhs, rhs)
    else:
        e_rows = np.linalg.norm(got_rows - ref_rows) / np.linalg.norm(ref_rows)
        e_frei = np.linalg.norm(lhs - rhs) / np.linalg.norm(rhs)
        assert e_rows <= TOL, e_rows
        assert e_frei <= TOL, e_frei
    torch.cuda.empty_cache()


def test_square_63360_bs64_densified(dbm, orc):
    run_and_check(dbm, orc, 63360, 63360, 63360, 64, "densified", 0)


def test_rect_bs64_densified(dbm, orc):
    run_and_check(dbm, orc, 1408, 1408, 1982464, 64, "densified", 0)


def test_rect_bs64_densified_integer_exact(dbm, orc):
    run_and_check(dbm, orc, 1408, 1408, 1982464, 64, "densified", 1)


def test_rect_bs22_blocked(dbm, orc):
    run_and_check(dbm, orc, 1408, 1408, 1982464, 22, "blocked", 0)


def test_square_63360_bs22_blocked_integer_exact(dbm, orc):
    run_and_check(dbm, orc, 63360, 63360, 63360, 22, "blocked", 1)
