"""NVLink byte counters of a Cannon-style copy-engine pull, through ncu's range replay (the pulls are DMA
copies, which ncu's kernel replay cannot attribute): GPU 0 pulls a 4 GiB panel from GPU 1 (1-D and 2-D
pitched copies, as dbm's pulls), alone and beside a persistent dbm GEMM on GPU 0, each inside a
cudaProfilerStart/Stop range.

    ncu --replay-mode app-range \
        --metrics nvlrx__bytes.sum,nvltx__bytes.sum,gpu__time_duration.sum --csv \
        python tools/microbench/nvlink_range.py
Without ncu it prints the pull rates (CUDA events).
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))


def cudart():
    """The CUDA runtime torch loaded (for cudaMemcpyPeerAsync: a copy-engine peer copy; torch's own
    cross-device copy_ may run as a kernel, which cannot start beside a persistent GEMM)."""
    import ctypes
    import glob

    import nvidia.cuda_runtime as cr

    lib = ctypes.CDLL(sorted(glob.glob(os.path.join(list(cr.__path__)[0], "lib", "libcudart.so*")))[0])
    lib.cudaMemcpyPeerAsync.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t,
                                        ctypes.c_void_p]
    return lib


def main():
    import paper_1910_04796_b200 as dbm

    rt = cudart()

    n = 1 << 29  # 4 GiB of doubles
    torch.cuda.set_device(0)
    src = torch.ones(n, dtype=torch.float64, device="cuda:1")
    dst = torch.empty(n, dtype=torch.float64, device="cuda:0")
    ctx = dbm.Context(device=0)
    M = N = K = 16384
    At = torch.rand(M, K, dtype=torch.float64, device="cuda:0")
    Bt = torch.rand(N, K, dtype=torch.float64, device="cuda:0")
    Cm = torch.empty(M * N, dtype=torch.float64, device="cuda:0")
    side = torch.cuda.Stream(device=0)
    for _ in range(2):  # warm-up (peer access, kernel load)
        dst.copy_(src)
        dbm.debug_dgemm(ctx, 2048, 2048, 2048, 1.0, At, K, Bt, K, 0.0, Cm, 2048)
    torch.cuda.synchronize(0)
    torch.cuda.synchronize(1)
    out = {}
    for name, with_gemm in (("pull_alone", False), ("pull_beside_gemm", True)):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.profiler.start()
        if with_gemm:
            dbm.debug_dgemm(ctx, M, N, K, 1.0, At, K, Bt, K, 0.0, Cm, M)  # persistent GEMM, every SM
        e0.record(side)
        r = rt.cudaMemcpyPeerAsync(dst.data_ptr(), 0, src.data_ptr(), 1, n * 8, side.cuda_stream)
        assert r == 0, r
        e1.record(side)
        torch.cuda.synchronize(0)
        torch.cuda.profiler.stop()
        ms = e0.elapsed_time(e1)
        out[name] = {"bytes": n * 8, "ms": ms, "gbs": n * 8 / ms / 1e6}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
