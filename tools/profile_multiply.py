"""Run dbm_multiply once or a few times at a given shape (single GPU), for ncu captures and quick timing.

    python tools/profile_multiply.py --M 5632 --N 5632 --K 5632 --bs 22 --path blocked --reps 2
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
    p.add_argument("--M", type=int, default=5632)
    p.add_argument("--N", type=int, default=5632)
    p.add_argument("--K", type=int, default=5632)
    p.add_argument("--bs", type=int, default=22)
    p.add_argument("--path", default="blocked")
    p.add_argument("--reps", type=int, default=2)
    p.add_argument("--occ", type=float, default=None, help="block occupancy of A and B (sparse, reading R15)")
    p.add_argument("--occ-c", type=float, default=1.0, help="block occupancy of C when --occ is given")
    a = p.parse_args()
    ctx = dbm.Context()
    if a.occ is None:
        A, B, C = dbm.Matrix(ctx, a.M, a.K, a.bs), dbm.Matrix(ctx, a.K, a.N, a.bs), dbm.Matrix(ctx, a.M, a.N, a.bs)
    else:
        Mb, Nb, Kb = a.M // a.bs, a.N // a.bs, a.K // a.bs
        A = dbm.Matrix(ctx, a.M, a.K, a.bs, mask=dbm.pattern_random(1910, 0, Mb, Kb, a.occ))
        B = dbm.Matrix(ctx, a.K, a.N, a.bs, mask=dbm.pattern_random(1910, 1, Kb, Nb, a.occ))
        C = dbm.Matrix(ctx, a.M, a.N, a.bs, mask=dbm.pattern_random(1910, 2, Mb, Nb, a.occ_c))
    A.fill_random(1910, 0, 0)
    B.fill_random(1910, 1, 0)
    C.fill_random(1910, 2, 0)
    for i in range(a.reps):
        ctx.set_profiling(i == a.reps - 1)  # phase times of the last repetition
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        st = dbm.multiply(ctx, 1.0, A, B, 0.0, C, a.path)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        ctx.set_profiling(False)
        phases = {n: ctx.profile_read(k)["ms"] for n, k in (("gemm", dbm.K_DGEMM), ("smm", dbm.K_SMM),
                                                             ("densify", dbm.K_DENSIFY), ("undensify", dbm.K_UNDENSIFY),
                                                             ("stackgen", dbm.K_STACKGEN))}
        eff = st["flops"] if a.occ is not None else 2.0 * a.M * a.N * a.K
        print(json.dumps({"M": a.M, "N": a.N, "K": a.K, "bs": a.bs, "path": a.path, "occ": a.occ, "rep": i, "ms": ms,
                          "tflops": eff / ms / 1e9, "entries": st["entries"], "stacks": st["stacks"],
                          "phases_ms": phases}), flush=True)


if __name__ == "__main__":
    main()
