"""Launch the densified path's FP64 GEMM (dbm_debug_dgemm) at a given shape, for ncu captures.

    python tools/profile_dgemm.py --M 63360 --N 63360 --K 15840 [--splitk 1] [--reps 2]

Default shape = one K-chunk GEMM of bench.py's default workload (63,360^3 bs 64, 1 GPU: four
63,360 x 63,360 x 15,840 launches per multiply).  Prints per-launch CUDA-event time and TFLOP/s.
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
    p.add_argument("--M", type=int, default=63360)
    p.add_argument("--N", type=int, default=63360)
    p.add_argument("--K", type=int, default=15840)
    p.add_argument("--splitk", type=int, default=0)
    p.add_argument("--reps", type=int, default=2)
    a = p.parse_args()
    M, N, K = a.M, a.N, a.K
    ld = K + (K % 2)
    ctx = dbm.Context()
    At = torch.rand(M, ld, dtype=torch.float64, device="cuda")
    Bt = torch.rand(N, ld, dtype=torch.float64, device="cuda")
    Cm = torch.empty(M * N, dtype=torch.float64, device="cuda")
    s = a.splitk
    part = torch.empty(max(s, 64) * M * N if (s != 1 and M * N < (1 << 26)) else 1, dtype=torch.float64,
                       device="cuda")
    for i in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        dbm.debug_dgemm(ctx, M, N, K, 1.0, At, ld, Bt, ld, 0.0, Cm, M, s, part)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        print(json.dumps({"M": M, "N": N, "K": K, "rep": i, "ms": ms, "tflops": 2.0 * M * N * K / ms / 1e9,
                          "algorithmic_bytes": 8.0 * (M * K + N * K + M * N)}), flush=True)


if __name__ == "__main__":
    main()
