"""Small multiplies that launch every kernel of the library once, for compute-sanitizer.

    compute-sanitizer --tool memcheck  python tools/sanitize_cases.py
    compute-sanitizer --tool racecheck python tools/sanitize_cases.py
    compute-sanitizer --tool synccheck python tools/sanitize_cases.py

Shapes are tiny (the sanitizers slow kernels by 10-100x) but each one reaches the kernel it names: the
dense DGEMM (densified path, bs 22 and zero-copy-B bs 64), the bs-22 square and group kernels, the bs-64
TMA kernel, the R x R run squares (DBM_SMMQ=2 forces them at small sizes), the per-size DMMA run kernels,
the FMA fallbacks, the block-sparse kernels (TMA-bulk bs 22, stream bs 64, run bs 5), the non-uniform
copy / pack / small-block kernels, the host-operand multiply. Prints one line per case; the sanitizer's
own summary is the result.
"""
import os
import sys

os.environ.setdefault("DBM_SMMQ", "2")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1910_04796_b200 as dbm  # noqa: E402


def run(ctx, name, A, B, C, path):
    A.fill_random(7, 0, 0)
    B.fill_random(7, 1, 0)
    C.fill_random(7, 2, 0)
    st = dbm.multiply(ctx, 0.75, A, B, -1.25, C, path)
    ctx.sync()
    print(name, path, st["entries"] if isinstance(st, dict) and "entries" in st else "", flush=True)


def main():
    ctx = dbm.Context()
    for M, N, K, bs in ((352, 352, 352, 22), (176, 88, 264, 22), (512, 512, 320, 64), (80 * 8, 80 * 8, 45, 5),
                        (72 * 8, 72 * 8, 36, 9), (130, 104, 169, 13), (96, 96, 128, 32), (70, 56, 49, 7)):
        for path in ("blocked", "densified"):
            run(ctx, f"dense {M}x{N}x{K} bs{bs}", dbm.Matrix(ctx, M, K, bs), dbm.Matrix(ctx, K, N, bs),
                dbm.Matrix(ctx, M, N, bs), path)
    for M, N, K, bs, occ in ((352, 352, 704, 22, 0.3), (512, 384, 640, 64, 0.4), (80, 60, 100, 5, 0.5)):
        Mb, Nb, Kb = M // bs, N // bs, K // bs
        for path in ("blocked", "densified"):
            A = dbm.Matrix(ctx, M, K, bs, mask=dbm.pattern_random(3, 0, Mb, Kb, occ))
            B = dbm.Matrix(ctx, K, N, bs, mask=dbm.pattern_random(3, 1, Kb, Nb, occ))
            C = dbm.Matrix(ctx, M, N, bs, mask=dbm.pattern_random(3, 2, Mb, Nb, 0.7))
            run(ctx, f"sparse {M}x{N}x{K} bs{bs}", A, B, C, path)
    rs, cs, ks = [5, 13, 23, 26, 13, 5, 32, 9], [13, 26, 5, 23, 9, 32], [23, 5, 26, 13, 32, 9, 5]
    for path in ("blocked", "densified"):
        A = dbm.Matrix(ctx, 0, 0, 0, row_sizes=rs, col_sizes=ks)
        B = dbm.Matrix(ctx, 0, 0, 0, row_sizes=ks, col_sizes=cs)
        C = dbm.Matrix(ctx, 0, 0, 0, row_sizes=rs, col_sizes=cs)
        run(ctx, "non-uniform cp2k mix", A, B, C, path)
    A, B, C = dbm.Matrix(ctx, 352, 352, 22), dbm.Matrix(ctx, 352, 352, 22), dbm.Matrix(ctx, 352, 352, 22)
    hosts = [torch.zeros(m.arena_bytes // 8, dtype=torch.float64, pin_memory=True) for m in (A, B, C)]
    for path in ("densified", "blocked"):
        dbm.multiply_host(ctx, 1.0, A, B, 0.0, C, *hosts, path=path)
        ctx.sync()
        print("host", path, flush=True)
    ctx.close()
    print("sanitize cases done")


if __name__ == "__main__":
    main()
