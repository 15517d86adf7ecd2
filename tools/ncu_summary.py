"""Summarise ncu outputs for profiles/ (run here, no GPU needed).

    python tools/ncu_summary.py launches <launches.csv>            # per-kernel share of device time
    python tools/ncu_summary.py full <report.ncu-rep> [algorithmic_bytes]   # key counters of a --set full capture
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

SCALE = {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3, "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0,
         "second": 1e3}

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor_subpipe_dmma.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "smsp__inst_executed_op_shared_ld.sum",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic", "sm__cycles_elapsed.avg.per_second",
        "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio"]


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    iname, ival, iunit = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot, cnt = defaultdict(float), defaultdict(int)
    for r in rows[1:]:
        name = r[iname].split("(")[0].replace("(anonymous namespace)::", "")
        tot[name] += float(r[ival].replace(",", "")) * SCALE[r[iunit]]
        cnt[name] += 1
    T = sum(tot.values())
    out = [{"kernel": n, "launches": cnt[n], "ms": round(tot[n], 3), "share": round(tot[n] / T, 5)}
           for n in sorted(tot, key=lambda x: -tot[x])]
    return {"total_ms": round(T, 3), "kernels": out}


def full(path, alg_bytes=None):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {"kernel": vals[hdr.index("Kernel Name")].split("(")[0].replace("(anonymous namespace)::", "")}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                d[k] = f"{vals[i]} {units[i]}".strip()
        res.append(d)
    if alg_bytes:
        for d in res:
            try:
                rd = d["dram__bytes_read.sum"].split()
                wr = d["dram__bytes_write.sum"].split()
                mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
                tb = float(rd[0].replace(",", "")) * mult[rd[1]] + float(wr[0].replace(",", "")) * mult[wr[1]]
                d["dram_traffic_bytes"] = tb
                d["algorithmic_bytes"] = float(alg_bytes)
                d["traffic_over_algorithmic"] = tb / float(alg_bytes)
            except Exception:
                pass
    return res


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    if mode == "launches":
        print(json.dumps(launches(path), indent=1))
    else:
        print(json.dumps(full(path, sys.argv[3] if len(sys.argv) > 3 else None), indent=1))
