"""Small-block GEMM comparison for §8f-4 (LIBCUSMM is 2-4x faster than cuBLAS batched DGEMM for
{m,n,k} < 32, saturating above 80): libdbm's blocked local multiply (stacks -> smm kernels) against
cuBLAS batched DGEMM (torch.matmul on the same block products, one batched call per inner block index
kk, batch = every C block), on one GPU.  cuBLAS is the comparison here, never on the product path.

    python tools/smm_vs_batched.py --n 5632 --bs 22 [--reps 3]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1910_04796_b200 as dbm  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--n", type=int, default=5632)
    p.add_argument("--bs", type=int, default=22)
    p.add_argument("--reps", type=int, default=3)
    a = p.parse_args()
    n, bs = a.n, a.bs
    nb = n // bs
    ctx = dbm.Context()
    A, B, C = dbm.Matrix(ctx, n, n, bs), dbm.Matrix(ctx, n, n, bs), dbm.Matrix(ctx, n, n, bs)
    A.fill_random(1910, 0, 0)
    B.fill_random(1910, 1, 0)
    flop = 2.0 * n * n * n
    ours = []
    for _ in range(a.reps + 1):
        ctx.set_profiling(True)
        dbm.multiply(ctx, 1.0, A, B, 0.0, C, "blocked")
        ctx.set_profiling(False)
        ours.append(ctx.profile_read(dbm.K_SMM)["ms"])
    # cuBLAS batched DGEMM with pointer arrays (cublasDgemmBatched, the P:187 comparison): for each inner
    # block index kk one call over every C block (li, lj): C_blk += A(li, kk) * B(kk, lj), beta = 1.
    import ctypes as ct

    import nvidia.cublas

    lib = ct.CDLL(os.path.join(list(nvidia.cublas.__path__)[0], "lib", "libcublas.so.12"))
    h = ct.c_void_p()
    assert lib.cublasCreate_v2(ct.byref(h)) == 0
    assert lib.cublasSetStream_v2(h, ct.c_void_p(torch.cuda.current_stream().cuda_stream)) == 0
    bb = bs * bs
    Cref = torch.zeros(nb * nb * bb, dtype=torch.float64, device="cuda")
    li = torch.arange(nb, device="cuda").repeat_interleave(nb)
    lj = torch.arange(nb, device="cuda").repeat(nb)
    base_a, base_b, base_c = A.arena.data_ptr(), B.arena.data_ptr(), Cref.data_ptr()
    carr = (base_c + (li * nb + lj) * bb * 8).to(torch.int64)
    arrs = []
    for kk in range(nb):  # pointer arrays built once (outside the timed region)
        aarr = (base_a + (li * nb + kk) * bb * 8).to(torch.int64)
        barr = (base_b + (kk * nb + lj) * bb * 8).to(torch.int64)
        arrs.append((aarr, barr))
    one = ct.c_double(1.0)
    f = lib.cublasDgemmBatched
    times = []
    for _ in range(a.reps + 1):
        Cref.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for aarr, barr in arrs:
            st = f(h, 0, 0, bs, bs, bs, ct.byref(one), ct.c_void_p(aarr.data_ptr()), bs, ct.c_void_p(barr.data_ptr()),
                   bs, ct.byref(one), ct.c_void_p(carr.data_ptr()), bs, nb * nb)
            assert st == 0, st
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    lib.cublasDestroy_v2(h)
    Cb = Cref.view(nb, nb, bs, bs).transpose(2, 3)
    got = C.arena[: nb * nb * bs * bs].view(nb, nb, bs, bs).transpose(2, 3)
    err = float((got - Cb).norm() / Cb.norm())
    t_ours, t_cub = min(ours[1:]), min(times[1:])
    print(json.dumps({"n": n, "bs": bs, "smm_ms": t_ours, "smm_tflops": flop / t_ours / 1e9,
                      "cublas_batched_ms": t_cub, "cublas_batched_tflops": flop / t_cub / 1e9,
                      "speedup": t_cub / t_ours, "relerr": err,
                      "note": "cublasDgemmBatched, one call of nb^2 block GEMMs per kk, beta = 1; ours = smm kernel "
                              "time of dbm_multiply (blocked)"}), flush=True)


if __name__ == "__main__":
    main()
