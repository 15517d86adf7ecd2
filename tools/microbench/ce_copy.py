"""Copy-engine transfer rates between two B200s over NVLink (and local), 1-D vs 2-D (pitched) copies:
the shapes the Cannon step-0 chunks and the tall-and-skinny gathers use.  Needs 2 GPUs.

    python tools/microbench/ce_copy.py
"""
import ctypes as ct
import json
import os

import torch

import nvidia.cuda_runtime

rt = ct.CDLL(os.path.join(list(nvidia.cuda_runtime.__path__)[0], "lib", "libcudart.so.12"))
D2D = 3


def timed(fn, stream, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    assert torch.cuda.device_count() >= 2
    torch.cuda.set_device(0)
    rows, pitch_el = 704, 495616 + 2  # a 2x2 rectangular-config panel: 704 rows, K-major
    src = torch.empty(rows * pitch_el, dtype=torch.float64, device="cuda:1")
    dst = torch.empty(rows * pitch_el, dtype=torch.float64, device="cuda:0")
    loc = torch.empty(rows * pitch_el, dtype=torch.float64, device="cuda:0")
    torch.cuda.synchronize()
    for d, o in ((0, 1), (1, 0)):  # direct NVLink peer access, as the library's IPC mappings have
        rt.cudaSetDevice(d)
        rt.cudaDeviceEnablePeerAccess(o, 0)
    rt.cudaSetDevice(0)
    rt.cudaGetLastError()
    s = torch.cuda.current_stream(0)
    sp = ct.c_void_p(s.cuda_stream)
    out = []
    for name, sbuf in (("peer", src), ("local", loc)):
        total = rows * pitch_el * 8
        ms = timed(lambda: rt.cudaMemcpyAsync(ct.c_void_p(dst.data_ptr()), ct.c_void_p(sbuf.data_ptr()),
                                              ct.c_size_t(total), D2D, sp), s)
        out.append({"src": name, "kind": "1d", "bytes": total, "ms": ms, "gbs": total / ms / 1e6})
        for frac in (1 / 16, 1 / 4, 1 / 2, 1.0):
            width = int(pitch_el * frac) // 2 * 2 * 8
            ms = timed(lambda: rt.cudaMemcpy2DAsync(ct.c_void_p(dst.data_ptr()), ct.c_size_t(pitch_el * 8),
                                                    ct.c_void_p(sbuf.data_ptr()), ct.c_size_t(pitch_el * 8),
                                                    ct.c_size_t(width), ct.c_size_t(rows), D2D, sp), s)
            out.append({"src": name, "kind": "2d", "rows": rows, "width_bytes": width, "bytes": width * rows, "ms": ms,
                        "gbs": width * rows / ms / 1e6})
    # the same copies while an FP64 GEMM occupies every SM on another stream (as in the Cannon pipeline)
    busy = torch.cuda.Stream(0)
    x = torch.randn(8192, 8192, dtype=torch.float64, device="cuda:0")
    for name, sbuf in (("peer", src), ("local", loc)):
        for kind, width in (("1d", None), ("2d", (pitch_el // 4) // 2 * 2 * 8)):
            nbytes = rows * pitch_el * 8 // 4 if kind == "1d" else width * rows
            def cp():
                if kind == "1d":
                    rt.cudaMemcpyAsync(ct.c_void_p(dst.data_ptr()), ct.c_void_p(sbuf.data_ptr()), ct.c_size_t(nbytes),
                                       D2D, sp)
                else:
                    rt.cudaMemcpy2DAsync(ct.c_void_p(dst.data_ptr()), ct.c_size_t(pitch_el * 8),
                                         ct.c_void_p(sbuf.data_ptr()), ct.c_size_t(pitch_el * 8), ct.c_size_t(width),
                                         ct.c_size_t(rows), D2D, sp)
            torch.cuda.synchronize()
            with torch.cuda.stream(busy):
                for _ in range(3):
                    y = x @ x  # ~90 ms of DGEMM
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            cp()
            e1.record(s)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            out.append({"src": name, "kind": kind, "under_gemm": True, "bytes": nbytes, "ms": ms, "gbs": nbytes / ms / 1e6})
            del y
    for o in out:
        print(json.dumps(o), flush=True)


if __name__ == "__main__":
    main()
