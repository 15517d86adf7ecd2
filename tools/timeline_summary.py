"""Summarise bench.py --timeline files: how much of each rank's Cannon pull time runs under its compute.

    python tools/timeline_summary.py profiles/r02/timelines/*.json

For every file: span (first start .. last end), compute time (dgemm / smm / densify / undensify / stackgen
records, merged intervals), pull time (merged pull intervals), the part of the pulls covered by compute,
and the compute-free part of the span (the exposed remainder: exposed pulls, waits, gaps).
"""
import json
import sys


def merge(iv):
    out = []
    for a, b in sorted(iv):
        if out and a <= out[-1][1]:
            out[-1][1] = max(out[-1][1], b)
        else:
            out.append([a, b])
    return out


def length(iv):
    return sum(b - a for a, b in iv)


def intersect(x, y):
    i = j = 0
    out = []
    while i < len(x) and j < len(y):
        a, b = max(x[i][0], y[j][0]), min(x[i][1], y[j][1])
        if a < b:
            out.append([a, b])
        if x[i][1] < y[j][1]:
            i += 1
        else:
            j += 1
    return out


def summary(path):
    d = json.load(open(path))
    rec = d["records"]
    if not rec:
        return None
    comp = merge([(r["start_ms"], r["end_ms"]) for r in rec if r["kind"] != "pull"])
    pull = merge([(r["start_ms"], r["end_ms"]) for r in rec if r["kind"] == "pull"])
    span = max(r["end_ms"] for r in rec) - min(r["start_ms"] for r in rec)
    covered = length(intersect(pull, comp))
    return {"file": path.split("/")[-1], "grid": d.get("grid"), "span_ms": round(span, 3),
            "compute_ms": round(length(comp), 3), "pull_ms": round(length(pull), 3),
            "pull_under_compute_ms": round(covered, 3),
            "pull_overlap": round(covered / length(pull), 4) if pull else None,
            "compute_free_ms": round(span - length(comp), 3)}


if __name__ == "__main__":
    for p in sys.argv[1:]:
        s = summary(p)
        if s:
            print(json.dumps(s))
