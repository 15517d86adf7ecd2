"""Benchmark: FP64 TFLOP/s of C = alpha*A*B + beta*C through libdbm (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config sq64|sq22|r64|r22|s352|sp22|sp64]
                    [--path densified|blocked] [--impl ours|reference]

A step is one dbm_multiply over the whole configuration (Cannon over the N-rank grid, every local
step, densify/undensify included).  N>1 runs under torchrun, one rank per GPU over NCCL.  Timing:
barrier + cuda synchronize on both sides of exactly K steps, CUDA events on the compute stream,
max over ranks.  Inputs are 8+ GB per matrix, far above the 126 MB L2, so no flush is needed.
Rank 0 prints one JSON line.  `--impl reference` times the host oracle (oracle/, test
infrastructure) on a bounded sample of the same workload instead.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "FP64 TFLOP/s per C=A·B (device-timed, max over ranks) at 1/2/4/8 B200; % of FP64 peak"
CONFIGS = {
    # name: (M, N, K, bs, default path, BASELINE.json configs[] index)
    "s352": (352, 352, 352, 22, "densified", 0),
    "sq64": (63360, 63360, 63360, 64, "densified", 1),
    "sq22": (63360, 63360, 63360, 22, "densified", 2),
    "r64": (1408, 1408, 1982464, 64, "densified", 3),
    "r22": (1408, 1408, 1982464, 22, "densified", 4),
    # block-sparse (§8f-2, reading R15; not a BASELINE config): A and B at 10 % block occupancy, C fully
    # stored; the metric counts only the stored block products (2 bs^3 per stack entry)
    "sp22": (63360, 63360, 63360, 22, "blocked", None),
    "sp64": (63360, 63360, 63360, 64, "blocked", None),
    # non-uniform block sizes (§8f-2 / f4, reading R16; not a BASELINE config): every dimension cut into
    # 1,000 blocks cycling through CP2K-like sizes 5, 13, 23, 26, 32 (19,800 elements)
    "nu": (19800, 19800, 19800, 0, "densified", None),
    "nus": (3960, 3960, 3960, 0, "densified", None),  # (the same at 200 blocks: profiling, quick A/B)
}
NU_CYCLE = (5, 13, 23, 26, 32)


def nu_sizes(total: int):
    out, i = [], 0
    while sum(out) < total:
        out.append(NU_CYCLE[i % len(NU_CYCLE)])
        i += 1
    assert sum(out) == total
    return out
SPARSE_OCC = {"sp22": (0.1, 0.1, 1.0), "sp64": (0.1, 0.1, 1.0)}
SEED = 1910
FP64_PEAK_MEASURED = 37.15  # TFLOP/s per B200, DMMA m8n8k4 chain at 1965 MHz (profiles/r01_fp64_peaks.jsonl)
FP64_PEAK_SPEC = 37.2       # 148 SM x 64 FMA/clk x 2 x 1.965 GHz


def _hbm_peak() -> float:
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6650.0  # fallback figure of the profiling guide


HBM_PEAK = _hbm_peak()


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=3)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--config", default="sq64", choices=sorted(CONFIGS))
    p.add_argument("--path", default=None, choices=["densified", "blocked", "auto"])
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--transport", default="ce", choices=["ce", "nccl"], help="Cannon panel transport (N>1)")
    p.add_argument("--grid", default="", help="force the process grid, e.g. 1x4 (default: reading R1)")
    p.add_argument("--algorithm", default="cannon", choices=["cannon", "tallskinny", "auto"],
                   help="MPI-level algorithm (P:168 Cannon / P:169 tall-and-skinny), N>1")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--e2e-steps", type=int, default=1)
    p.add_argument("--timeline", default="", help="write one profiled multiply's per-rank timeline "
                   "(kernels on every stream and the Cannon pulls, CUDA events) to <path>.rank<r>.json")
    return p.parse_args()


# ------------------------------------------------------------------ clocks during the timed region
class ClockSampler:
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, device: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ------------------------------------------------------------------ reference arm / cpu baseline
CPU_ROWS = 64  # the oracle is timed on the verification workload's 64 sampled rows of C


def _sample_rows(M: int):
    import numpy as np

    return np.linspace(0, M - 1, min(CPU_ROWS, M)).astype(np.int64)


def oracle_sample(M, N, K, bs, kpre: int, occ=None) -> dict:
    """Time the host oracle, as it stands, on a fixed sample of the workload: the same 64 rows of C
     over the first `kpre` columns of A / rows of B (whole blocks).  The oracle's cost is
    the same per (k, j) pair for a fixed row set, so the rate does not depend on kpre and every sample
    of a config measures the same thing; `extrapolated_full_s` = t * (M / 64) * (K / kpre)."""
    import oracle

    oracle.build()
    idx = _sample_rows(M)
    t0 = time.perf_counter()
    if occ:
        _, fmas = oracle.sparse_rows_from_seeds(M, N, kpre, bs, SEED, 0, SEED, occ[0], occ[1], occ[2], 1.0, 0.0, idx)
        flop = 2.0 * fmas
    else:
        oracle.rows_from_seeds(M, N, kpre, SEED, 0, 1.0, 0.0, idx)
        flop = 2.0 * len(idx) * kpre * N
    dt = time.perf_counter() - t0
    full = dt * (M / len(idx)) * (K / kpre)
    what = "block-sparse C (useful flop)" if occ else "C = A*B"
    return {"value": flop / dt / 1e12, "unit": "TFLOP/s", "cores": oracle.num_threads(), "kind": "oracle",
            "sample": f"rows {len(idx)} of {M} (np.linspace) x k < {kpre} of {K} of {what} regenerated from seeds "
                      f"({flop:.3g} flop, {dt:.2f} s)",
            "extrapolated_full_s": full, "extrapolated": True, "seconds": dt}


def oracle_kpre(M, N, K, bs, target_s: float, occ=None) -> int:
    """K prefix (whole blocks) that makes one 64-row sample take about target_s on this host: one short
    probe on the same rows, then linear scaling (the oracle's time is linear in the K prefix)."""
    bs = bs or 1  # non-uniform blocks: the oracle's rows do not depend on the blocking
    probe_k = min(K, bs * max(1, -(-256 // bs)))
    t = oracle_sample(M, N, K, bs, probe_k, occ)["seconds"]
    k = int(probe_k * target_s / max(t, 1e-4)) // bs * bs
    return max(bs, min(K, k))


def run_reference(args, cfg, name, world, rank):
    M, N, K, bs, path, _ = cfg
    if rank != 0:
        return
    if world > 1 and os.environ.get("OMP_NUM_THREADS") == "1":
        # torchrun pins every process to one OpenMP thread; rank 0 is the only one working here, so it
        # gets the host's cores, as at N = 1 (set before the oracle library, and its OpenMP, load)
        os.environ["OMP_NUM_THREADS"] = str(len(os.sched_getaffinity(0)))
    occ = SPARSE_OCC.get(args.config)
    kpre = oracle_kpre(M, N, K, bs, 4.0, occ)  # each step: the fixed 64-row sample over a K prefix (~4 s)
    times = []
    for i in range(args.warmup + args.steps):
        r = oracle_sample(M, N, K, bs, kpre, occ)
        if i >= args.warmup:
            times.append(r)
    val = statistics.mean(t["value"] for t in times)
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "TFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": statistics.mean(t["seconds"] for t in times) * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": name, "M": M, "N": N, "K": K, "block_size": bs, "path": path},
        "cpu_baseline": {k: times[-1][k] for k in ("kind", "cores", "sample", "extrapolated_full_s", "extrapolated")}
        | {"value": val, "unit": "TFLOP/s"},
        "e2e": {"value": val, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(line)


_OUT = None  # the stream the ONE JSON line goes to (set in __main__)


def emit(line):
    """Print the bench's single JSON line on the real stdout (everything else, including native
    libraries' stdout chatter such as NCCL's version banner, is redirected to stderr)."""
    out = _OUT or sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()


# ------------------------------------------------------------------ our arm
def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    cfg = CONFIGS[args.config]
    M, N, K, bs, dpath, cidx = cfg
    path = args.path or dpath
    name = {"s352": "352^3 bs22", "sq64": "square 63360^3 bs64", "sq22": "square 63360^3 bs22",
            "r64": "rect 1408x1408x1982464 bs64", "r22": "rect 1408x1408x1982464 bs22",
            "sp22": "square 63360^3 bs22 block-sparse A,B occupancy 0.1, C stored",
            "sp64": "square 63360^3 bs64 block-sparse A,B occupancy 0.1, C stored",
            "nu": "square 19800^3 non-uniform blocks cycling 5,13,23,26,32",
            "nus": "square 3960^3 non-uniform blocks cycling 5,13,23,26,32"}[args.config]
    occ = SPARSE_OCC.get(args.config)
    name = f"{name} {path} " + (f"(BASELINE.json configs[{cidx}])" if cidx is not None else "(§8f-2 NEXT row)")
    if args.impl == "reference":
        return run_reference(args, (M, N, K, bs, path, cidx), name, world, rank)

    import torch
    import torch.distributed as dist

    import paper_1910_04796_b200 as dbm

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        pr, pc = (int(x) for x in args.grid.split("x")) if args.grid else (0, 0)
        ctx = dbm.Context.from_distributed(pr=pr, pc=pc)
        ctx.set_transport(args.transport)
        ctx.set_algorithm(args.algorithm)
    else:
        ctx = dbm.Context(device=local)
    stream = torch.cuda.current_stream(dev)
    if occ:
        Mb, Nb, Kb = M // bs, N // bs, K // bs
        A = dbm.Matrix(ctx, M, K, bs, mask=dbm.pattern_random(SEED, 0, Mb, Kb, occ[0]))
        B = dbm.Matrix(ctx, K, N, bs, mask=dbm.pattern_random(SEED, 1, Kb, Nb, occ[1]))
        C = dbm.Matrix(ctx, M, N, bs, mask=dbm.pattern_random(SEED, 2, Mb, Nb, occ[2]))
    elif bs == 0:  # non-uniform block sizes
        ms, ns, ks = nu_sizes(M), nu_sizes(N), nu_sizes(K)
        A = dbm.Matrix(ctx, 0, 0, 0, row_sizes=ms, col_sizes=ks)
        B = dbm.Matrix(ctx, 0, 0, 0, row_sizes=ks, col_sizes=ns)
        C = dbm.Matrix(ctx, 0, 0, 0, row_sizes=ms, col_sizes=ns)
    else:
        A, B, C = dbm.Matrix(ctx, M, K, bs), dbm.Matrix(ctx, K, N, bs), dbm.Matrix(ctx, M, N, bs)
    A.fill_random(SEED, 0, 0)
    B.fill_random(SEED, 1, 0)
    C.fill_random(SEED, 2, 0)
    ws = ctx.workspace(dbm.multiply_workspace(ctx, A, B, C, path))
    alpha, beta = 1.0, 0.0

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local])
        torch.cuda.synchronize()

    def maxrank(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(args.warmup):
        dbm.multiply(ctx, alpha, A, B, beta, C, path, workspace=ws)
    barrier()
    launches0 = ctx.launch_count()
    ctx.set_profiling(True)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    host_ms = []
    with ClockSampler(local) as clk:
        barrier()
        ev0.record(stream)
        evs[0].record(stream)
        for i in range(args.steps):
            h0 = time.perf_counter()
            st = dbm.multiply(ctx, alpha, A, B, beta, C, path, workspace=ws)
            host_ms.append((time.perf_counter() - h0) * 1e3)  # host enqueue time of the call
            evs[i + 1].record(stream)
        ev1.record(stream)
        barrier()
    ctx.set_profiling(False)
    launches = ctx.launch_count() - launches0
    ms = maxrank(ev0.elapsed_time(ev1)) / args.steps
    flop = 2.0 * M * N * K
    if occ:  # useful flops of the stored block products, summed over ranks
        flop = st["flops"]
        if world > 1:
            t = torch.tensor([flop], dtype=torch.float64, device=dev)
            dist.all_reduce(t)
            flop = float(t.item())
    tflops = flop / (ms * 1e-3) / 1e12
    kern = "dgemm" if path == "densified" else "smm"
    prof = ctx.profile_read(dbm.K_DGEMM if path == "densified" else dbm.K_SMM)
    prof_d = ctx.profile_read(dbm.K_DENSIFY)
    prof_u = ctx.profile_read(dbm.K_UNDENSIFY)
    prof_s = ctx.profile_read(dbm.K_STACKGEN)
    prof_x = ctx.profile_read(dbm.K_EXCHANGE)
    per_launch_ms = prof["ms"] / max(prof["launches"], 1)
    per_launch_flop = prof["flops"] / max(prof["launches"], 1)
    achieved = per_launch_flop / (per_launch_ms * 1e-3) / 1e12 if per_launch_ms > 0 else None
    traffic = None
    tfile = os.path.join(ROOT, "profiles", f"traffic_{args.config}_{path}_n{world}.json")
    if os.path.exists(tfile):
        traffic = json.load(open(tfile)).get("bytes_per_launch")

    if args.timeline:  # one more multiply with every record kept: the overlap of pulls and GEMMs
        write_timeline(args, ctx, dbm, lambda: dbm.multiply(ctx, alpha, A, B, beta, C, path, workspace=ws),
                       args.timeline, name)

    # ---------------- end to end through the public API with host buffers (pinned), rank-local shares
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, ctx, dbm, torch, A, B, C, path, ws, stream, barrier, maxrank, flop)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:  # the same fixed 64-row sample as the reference arm, over a K prefix sized to ~15 s
            cpu = oracle_sample(M, N, K, bs, oracle_kpre(M, N, K, bs, 15.0, occ), occ)
            cpu.pop("seconds", None)
        except Exception as ex:  # reported, never fatal
            cpu = {"error": str(ex)[:200]}

    if rank == 0:
        line = {
            "metric": METRIC, "value": tflops, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": name, "M": M, "N": N, "K": K, "block_size": bs, "path": path,
                       "grid": f"{ctx.pr}x{ctx.pc}", "parallelism": f"cannon{ctx.pr}x{ctx.pc}",
                       "transport": (args.transport if world > 1 else None),
                       "algorithm": (args.algorithm if world > 1 else "local"),
                       "l2": ("inputs 3.1 GB per matrix >> 126 MB L2; no flush" if bs == 0 else
                              "inputs >= 8 GB per matrix >> 126 MB L2; no flush" if not occ else
                              "A, B 3.2 GB each (10 % of 32 GB) >> 126 MB L2; no flush"), "alpha": alpha, "beta": beta,
                       "occupancy": occ},
            "pct_fp64_peak": 100.0 * tflops / (world * FP64_PEAK_MEASURED),
            "roofline": {"kernel": kern, "bound": "tensor", "achieved": achieved, "peak": FP64_PEAK_MEASURED,
                         "unit": "TFLOP/s", "frac": (achieved / FP64_PEAK_MEASURED) if achieved else None,
                         "traffic": traffic, "launches": prof["launches"], "ms_per_launch": per_launch_ms,
                         "flop_per_launch": per_launch_flop,
                         "peak_source": "measured FP64 DMMA peak, profiles/r01_fp64_peaks.jsonl (FP64 is not in "
                                        "MEASURED_PEAKS.json); spec 37.2",
                         "share_of_step": prof["ms"] / (ms * args.steps) if ms > 0 else None},
            "phases_ms_per_step": {"dgemm_or_smm": prof["ms"] / args.steps, "densify": prof_d["ms"] / args.steps,
                                   "undensify": prof_u["ms"] / args.steps, "stackgen": prof_s["ms"] / args.steps},
            # HBM-bound kernels of the path: algorithmic bytes / CUDA-event time vs the measured copy peak
            "hbm_kernels": {name: {"gbs": (pr_["bytes"] / (pr_["ms"] * 1e-3) / 1e9) if pr_["ms"] > 0 else None,
                                   "frac": (pr_["bytes"] / (pr_["ms"] * 1e-3) / 1e9 / HBM_PEAK) if pr_["ms"] > 0
                                   else None, "launches": pr_["launches"]}
                            for name, pr_ in (("densify", prof_d), ("undensify", prof_u), ("stackgen", prof_s))
                            if pr_["launches"]},
            "stats": {k: st[k] for k in ("entries", "stacks", "bytes_sent", "bytes_recv", "steps")},
            # Cannon transport (rank 0): copy-engine pull time on the comm stream, bytes received, the
            # achieved NVLink rate, and the step time not covered by the rank's kernels (exposed comm +
            # barriers + gaps) = ms_per_step - sum of the phases above
            "exchange": ({"ms_per_step": prof_x["ms"] / args.steps, "bytes_per_step": prof_x["bytes"] / args.steps,
                          "gbs": prof_x["bytes"] / (prof_x["ms"] * 1e-3) / 1e9 if prof_x["ms"] > 0 else None,
                          "uncovered_ms_per_step": ms - (prof["ms"] + prof_d["ms"] + prof_u["ms"] + prof_s["ms"])
                          / args.steps} if world > 1 else None),
            # rank 0: device time of every timed step (CUDA events between the calls) and the host time each
            # call took to enqueue (the call returns before its work runs; a host slower than the device
            # would show as gaps between steps)
            "steps_ms": [evs[i].elapsed_time(evs[i + 1]) for i in range(args.steps)],
            "host_enqueue_ms": host_ms,
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        emit(line)
    if world > 1:
        dist.barrier(device_ids=[local])
        dist.destroy_process_group()


def write_timeline(args, ctx, dbm, call, prefix, name=""):
    """Run `call` once with profiling on; write its records (kind, start, end in ms, CUDA events on every
    stream the library uses) to <prefix>.rank<r>.json."""
    ctx.sync()
    ctx.set_profiling(True)
    call()  # two calls back to back, as in the timed loop: the gap between them is part of the record
    call()
    ctx.sync()
    names = {dbm.K_DGEMM: "dgemm", dbm.K_SMM: "smm", dbm.K_DENSIFY: "densify", dbm.K_UNDENSIFY: "undensify",
             dbm.K_STACKGEN: "stackgen", dbm.K_EXCHANGE: "pull"}
    tl = [{"kind": names.get(k, k), "start_ms": a, "end_ms": b} for k, a, b in ctx.profile_timeline()]
    ctx.set_profiling(False)
    for k in names:
        ctx.profile_read(k)  # drop the records
    with open(f"{prefix}.rank{ctx.rank}.json", "w") as fh:
        json.dump({"rank": ctx.rank, "grid": f"{ctx.pr}x{ctx.pc}", "config": name or args.config, "records": tl}, fh,
                  indent=0)


def run_e2e(args, ctx, dbm, torch, A, B, C, path, ws, stream, barrier, maxrank, flop):
    """Same metric through the public C-ABI call with HOST buffers (dbm_multiply_host): per step the H2D
    of A and B from pinned host memory (streamed in K-chunks under the GEMMs on one GPU), the multiply
    and the D2H of C (beta = 0, so C_in is not read: BLAS convention, reading R8)."""
    try:
        hA = torch.empty(A.arena_bytes // 8, dtype=torch.float64, pin_memory=True)
        hB = torch.empty(B.arena_bytes // 8, dtype=torch.float64, pin_memory=True)
        hC = torch.empty(C.arena_bytes // 8, dtype=torch.float64, pin_memory=True)
        pinned = True
    except Exception:
        hA = torch.empty(A.arena_bytes // 8, dtype=torch.float64)
        hB = torch.empty(B.arena_bytes // 8, dtype=torch.float64)
        hC = torch.empty(C.arena_bytes // 8, dtype=torch.float64)
        pinned = False
    A.download(hA)
    B.download(hB)
    ctx.sync()

    def step():  # one C-ABI call with host buffers (dbm_multiply_host: streamed H2D, D2H of C)
        dbm.multiply_host(ctx, 1.0, A, B, 0.0, C, hA, hB, hC, path, workspace=ws)

    step()  # warm-up
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.e2e_steps):
        step()
    e1.record(stream)
    barrier()
    ms = maxrank(e0.elapsed_time(e1)) / args.e2e_steps
    if args.timeline:  # one more profiled host-operand multiply (uploads, own-panel chunks, pulls, GEMMs)
        write_timeline(args, ctx, dbm, step, f"{args.timeline}.e2e")
    out = {"value": flop / (ms * 1e-3) / 1e12, "unit": "TFLOP/s", "h2d_bytes_per_step": A.arena_bytes + B.arena_bytes,
           "d2h_bytes_per_step": C.arena_bytes, "ms_per_step": ms, "steps": args.e2e_steps,
           "host_memory": "pinned" if pinned else "pageable (staged through libdbm's pinned double buffer)",
           "bytes_are": "rank-local shares (rank 0 shown)"}
    del hA, hB, hC
    return out


if __name__ == "__main__":
    # keep stdout to exactly one JSON line: the real stdout is kept for emit(), fd 1 (which native
    # code such as NCCL prints to) goes to stderr
    sys.stdout.flush()
    _OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    main()
