"""Run every BASELINE.json config through bench.py and print the report table (markdown + JSON).

    python tools/report.py [--gpus N] [--steps K] [--warmup W] [--out profiles/report.json]

Per config: TFLOP/s, % of FP64 peak (N x 37.15 measured), dominant-kernel roofline fraction, and the
blocked/densified time ratio per block size (the paper's Fig. 3 quantity, §IV.B).  The
paper's own numbers are relative only and are quoted as context.
N > 1 runs each bench under torch.distributed.run on this node.
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

RUNS = [("s352", "densified"), ("s352", "blocked"), ("sq64", "densified"), ("sq64", "blocked"),
        ("sq22", "densified"), ("sq22", "blocked"), ("r64", "densified"), ("r64", "blocked"),
        ("r22", "densified"), ("r22", "blocked")]
PAPER = {
    "sq": "densified up to 80% faster than blocked (T_blocked/T_densified <= 1.8), gain shrinking with node count (P:49)",
    "r": "smaller gain, limited by densify/undensify overhead (P:52)",
}


def run(cfg, path, gpus, steps, warmup, port):
    base = [sys.executable]
    if gpus > 1:
        base += ["-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}", "--master-addr=127.0.0.1",
                 f"--master-port={port}"]
    cmd = base + [os.path.join(ROOT, "bench.py"), "--gpus", str(gpus), "--config", cfg, "--path", path,
                  "--steps", str(steps), "--warmup", str(warmup), "--no-e2e", "--no-cpu-baseline"]
    r = subprocess.run(cmd, capture_output=True, text=True, cwd=ROOT)
    for line in r.stdout.splitlines():
        if line.startswith("{"):
            return json.loads(line)
    return {"error": (r.stderr or r.stdout)[-400:]}


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=2)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--only", default="")
    p.add_argument("--out", default="")
    a = p.parse_args()
    res = {}
    for i, (cfg, path) in enumerate(RUNS):
        if a.only and cfg not in a.only.split(","):
            continue
        d = run(cfg, path, a.gpus, a.steps, a.warmup, 29600 + i)
        res[f"{cfg}/{path}"] = d
        print(json.dumps({"run": f"{cfg}/{path}", "value": d.get("value"), "ms": d.get("ms_per_step"),
                          "error": d.get("error")}), flush=True)
    rows = ["| config | path | ms / multiply | TFLOP/s | % FP64 peak | kernel | kernel frac | T_blocked/T_densified |",
            "|---|---|---|---|---|---|---|---|"]
    for cfg in ("s352", "sq64", "sq22", "r64", "r22"):
        dd, db = res.get(f"{cfg}/densified", {}), res.get(f"{cfg}/blocked", {})
        ratio = (db["ms_per_step"] / dd["ms_per_step"]) if ("ms_per_step" in dd and "ms_per_step" in db) else None
        for path, d in (("densified", dd), ("blocked", db)):
            if "value" not in d:
                continue
            rf = d.get("roofline", {})
            rows.append(f"| {cfg} | {path} | {d['ms_per_step']:.2f} | {d['value']:.2f} | {d['pct_fp64_peak']:.1f} | "
                        f"{rf.get('kernel')} | {rf.get('frac') or 0:.3f} | "
                        f"{'' if path == 'densified' or ratio is None else f'{ratio:.2f}'} |")
    table = "\n".join(rows)
    print(table)
    if a.out:
        json.dump({"gpus": a.gpus, "results": res, "table_md": table, "paper_context": PAPER}, open(a.out, "w"),
                  indent=1)


if __name__ == "__main__":
    main()
