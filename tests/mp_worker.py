"""torchrun worker for tests/test_multigpu.py: multi-rank parity of dbm_multiply over NCCL.

For every factorisation pr x pc of the world size, both local paths and several (ragged) shapes:
fill A, B, C per rank, multiply, compare the rank's share with the oracle's product scattered to
that rank (normwise relative error <= 1e-12; bit-exact for integer inputs), and the rank's Cannon
bytes with the oracle's schedule.  Exits non-zero on any failure; rank 0 prints one JSON per case.
"""
import argparse
import faulthandler
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle as orc  # noqa: E402  (test infrastructure)
import paper_1910_04796_b200 as dbm  # noqa: E402

SEED = 1910


class Watchdog:
    """Per-case hang guard: a case that does not finish within `seconds` dumps every thread's Python
    stack and exits the process non-zero (torchrun then tears the other ranks down), so one hung
    multiply fails one test run quickly instead of stalling the suite."""

    def __init__(self, seconds: float):
        self.seconds = seconds

    def __enter__(self):
        faulthandler.dump_traceback_later(self.seconds, exit=True)
        return self

    def __exit__(self, *a):
        faulthandler.cancel_dump_traceback_later()


CASE_TIMEOUT = float(os.environ.get("DBM_CASE_TIMEOUT", "120"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--groups", default="cannon,sparse,host,sweep,nonuni",
                    help="comma list of case groups: cannon, sparse, host, sweep, nonuni")
    ap.add_argument("--summary", default="", help="rank 0 writes a JSON summary here")
    args = ap.parse_args()
    groups = set(args.groups.split(","))
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    world, rank = dist.get_world_size(), dist.get_rank()
    grids = [(p, world // p) for p in range(1, world + 1) if world % p == 0]
    summary = {"world": world, "grids": [f"{a}x{b}" for a, b in grids], "groups": {}}
    failures = 0
    if "cannon" in groups:
        f, n, e = cannon_cases(world, rank, dev, grids)
        summary["groups"]["cannon"] = {"cases": n, "failures": f, "max_err": e}
        failures += f
    if "sparse" in groups:
        f, n, e = sparse_cases(world, rank, dev, grids)
        summary["groups"]["sparse"] = {"cases": n, "failures": f, "max_err": e}
        failures += f
    if "host" in groups:
        f, n = host_cases(world, rank, dev, grids, HOST_SHAPES)
        summary["groups"]["host"] = {"cases": n, "failures": f}
        failures += f
    if "nonuni" in groups:
        f, n, e = nonuni_cases(world, rank, dev, grids)
        summary["groups"]["nonuni"] = {"cases": n, "failures": f, "max_err": e}
        failures += f
    if "sweep" in groups:
        f, n = host_cases(world, rank, dev, grids, sweep_shapes())
        summary["groups"]["host_sweep"] = {"cases": n, "failures": f}
        failures += f
    summary["failures"] = failures
    if rank == 0:
        print(json.dumps({"summary": summary}), flush=True)
        if args.summary:
            with open(args.summary, "w") as fh:
                json.dump(summary, fh, indent=1)
    dist.barrier(device_ids=[local])
    dist.destroy_process_group()
    sys.exit(1 if failures else 0)


def cannon_cases(world, rank, dev, grids):
    """Device-resident multiply on every grid, both transports and algorithms, both paths."""
    shapes = [(352, 352, 352, 22), (704, 528, 1100, 22), (384, 640, 1280, 64), (66, 154, 198, 22), (44, 44, 22, 22)]
    failures = ncases = 0
    max_err = 0.0
    cases = [(pr, pc, tr, "cannon") for (pr, pc) in grids for tr in ("ce", "nccl")]
    cases += [(pr, pc, "ce", "tallskinny") for (pr, pc) in grids]
    cases += [(pr, pc, "ce", "auto") for (pr, pc) in grids]  # tall-and-skinny iff K >= 16 max(M, N)
    for pr, pc, transport, algo in cases:
        ctx = dbm.Context.from_distributed(pr=pr, pc=pc)
        ctx.set_transport(transport)
        ctx.set_algorithm(algo)
        r, c = ctx.myrow, ctx.mycol
        for (M, N, K, bs) in (shapes + [(88, 66, 2816, 22)] if algo == "auto" else shapes):
            for path in (("densified",) if algo == "tallskinny" else ("densified", "blocked")):
                for kind in (0, 1):
                    A, B, C = dbm.Matrix(ctx, M, K, bs), dbm.Matrix(ctx, K, N, bs), dbm.Matrix(ctx, M, N, bs)
                    A.fill_random(SEED, 0, kind)
                    B.fill_random(SEED, 1, kind)
                    C.fill_random(SEED, 2, kind)
                    with Watchdog(CASE_TIMEOUT):
                        for rep in range(2):  # second call reuses the workspace / exchange buffers
                            if rep == 1:
                                C.fill_random(SEED, 2, kind)
                            st = dbm.multiply(ctx, 0.75, A, B, -1.25, C, path)
                        torch.cuda.synchronize()
                    got = C.arena.cpu().numpy()[: C.arena_bytes // 8]
                    Ag = orc.fill_arena(SEED, 0, kind, M, K, bs)
                    Bg = orc.fill_arena(SEED, 1, kind, K, N, bs)
                    Cg = orc.fill_arena(SEED, 2, kind, M, N, bs)
                    orc.multiply_blocked(M // bs, N // bs, K // bs, bs, 0.75, Ag, Bg, -1.25, Cg)
                    ref = orc.scatter(Cg, M // bs, N // bs, bs, pr, pc, r, c)
                    if kind == 1:
                        ok_val = np.array_equal(got, ref)
                        err = float(np.abs(got - ref).max()) if ref.size else 0.0
                    else:
                        err = float(np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-300)) if ref.size else 0.0
                        ok_val = err <= 1e-12
                    ts = algo == "tallskinny" or (algo == "auto" and path == "densified" and K >= 16 * max(M, N))
                    if not ts:
                        rv, sd = orc.cannon_bytes(M // bs, N // bs, K // bs, bs, pr, pc, r, c)
                    else:
                        rv, sd = orc.ts_bytes(M // bs, N // bs, K // bs, bs, pr, pc, r, c)
                    ok_bytes = (st["bytes_recv"], st["bytes_sent"]) == (rv, sd)
                    flags = torch.tensor([0 if (ok_val and ok_bytes) else 1], device=dev)
                    dist.all_reduce(flags)
                    ncases += 1
                    max_err = max(max_err, err)
                    if flags.item():
                        failures += 1
                    if rank == 0 or not (ok_val and ok_bytes):
                        print(json.dumps({"rank": rank, "grid": f"{pr}x{pc}", "transport": transport, "algo": algo, "shape": [M, N, K, bs], "path": path,
                                          "kind": kind, "err": err, "ok": bool(ok_val), "bytes_ok": ok_bytes,
                                          "recv": st["bytes_recv"], "expect_recv": rv}), flush=True)
        ctx.close()
    return failures, ncases, max_err


# dbm_multiply_host on several ranks: (M, N, K, bs, beta, path).  The 352^3 bs-22 beta = 0 cases are the
# round-1 bench hang (1 x 2 grid, 8-block panels); bs 13 / 9 are odd block sizes (odd bs^2: blocks
# alternate 8 mod 16 byte alignment, odd bs: dense panel columns too).
HOST_SHAPES = [(352, 352, 704, 22, -1.25, "densified"), (320, 192, 640, 64, 0.0, "densified"),
               (198, 154, 330, 22, 1.0, "densified"), (352, 352, 704, 22, -1.25, "blocked"),
               (198, 154, 330, 22, 1.0, "blocked"), (320, 192, 640, 64, 0.0, "blocked"),
               (352, 352, 352, 22, 0.0, "densified"), (352, 352, 352, 22, 0.0, "blocked"),
               (130, 104, 416, 13, 0.0, "blocked"), (130, 104, 416, 13, -1.25, "densified"),
               (117, 90, 243, 9, 1.0, "blocked"), (117, 90, 243, 9, 0.0, "densified")]


def sweep_shapes():
    """Panel block counts 1..16 on the widest grid (K = 4 kb blocks covers L <= 4), both betas, both
    paths, bs 22 and 64: every pattern of empty / non-empty host-pipeline chunks."""
    out = []
    for kb in range(1, 17):
        for bs in (22, 64):
            for beta in (0.0, -1.25):
                for path in ("densified", "blocked"):
                    out.append((4 * bs, 2 * bs, 4 * kb * bs, bs, beta, path))
    return out


def host_cases(world, rank, dev, grids, shapes):
    """dbm_multiply_host on every grid (pinned host arenas; the last GEMM's row panels are downloaded while
    the next multiplies): C_host against the oracle, float and integer inputs.
    Several ranks: uploads, own-panel densify and the step-0 pull + GEMM run in 5 K-chunks gated by the
    owners' published progress (ragged K: empty first chunks; bs 64: packed zero-copy B panels); the
    blocked path packs its own panels chunk by chunk the same way, C_in uploaded first."""
    failures = ncases = 0
    for pr, pc in grids:
        ctx = dbm.Context.from_distributed(pr=pr, pc=pc)
        r, c = ctx.myrow, ctx.mycol
        for (M, N, K, bs, beta, path), kind in [(sh, kd) for sh in shapes for kd in (0, 1)]:
            A, B, C = dbm.Matrix(ctx, M, K, bs), dbm.Matrix(ctx, K, N, bs), dbm.Matrix(ctx, M, N, bs)
            hs = []
            for m, mid in ((A, 0), (B, 1), (C, 2)):
                m.fill_random(SEED, mid, kind)
                h = torch.empty(max(m.arena_bytes // 8, 1), dtype=torch.float64, pin_memory=True)
                m.download(h)
                hs.append(h)
            ctx.sync()
            for m in (A, B, C):
                m.arena.zero_()  # the device copies are only staging: results must come from the host buffers
            with Watchdog(CASE_TIMEOUT):
                dbm.multiply_host(ctx, 0.75, A, B, beta, C, hs[0], hs[1], hs[2], path)
                ctx.sync()
            got = hs[2].numpy()[: C.arena_bytes // 8]
            Ag = orc.fill_arena(SEED, 0, kind, M, K, bs)
            Bg = orc.fill_arena(SEED, 1, kind, K, N, bs)
            Cg = orc.fill_arena(SEED, 2, kind, M, N, bs)
            orc.multiply_blocked(M // bs, N // bs, K // bs, bs, 0.75, Ag, Bg, beta, Cg)
            ref = orc.scatter(Cg, M // bs, N // bs, bs, pr, pc, r, c)
            ok = np.array_equal(got, ref) if kind == 1 else \
                float(np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-300)) <= 1e-12
            flags = torch.tensor([0 if ok else 1], device=dev)
            dist.all_reduce(flags)
            failures += int(flags.item() > 0)
            ncases += 1
            if (rank == 0 and shapes is HOST_SHAPES) or not ok:
                print(json.dumps({"rank": rank, "grid": f"{pr}x{pc}", "host": True, "shape": [M, N, K, bs], "path": path,
                                  "beta": beta, "kind": kind, "ok": bool(ok)}),
                      flush=True)
        ctx.close()
    return failures, ncases


def nonuni_cases(world, rank, dev, grids):
    """Non-uniform block sizes (reading R16) on every grid: both paths (densified also block-sparse),
    float <= 1e-12 and integer bit-exact against orc_nu_multiply scattered to this rank."""
    failures = ncases = 0
    max_err = 0.0
    mixes = [([5, 13, 23, 26, 13, 5, 32, 9, 22], [13, 26, 5, 23, 9, 32, 7], [23, 5, 26, 13, 32, 9, 5, 11, 4]),
             ([22, 64, 22, 64, 22], [64, 22, 64, 22], [22, 22, 64, 64, 22, 64, 22])]
    for pr, pc in grids:
        ctx = dbm.Context.from_distributed(pr=pr, pc=pc)
        r, c = ctx.myrow, ctx.mycol
        for mi, (ms, ns, ks) in enumerate(mixes):
            for path, sparse in (("densified", False), ("blocked", False), ("densified", True)):
                masks = (orc.pattern_random(4, 0, len(ms), len(ks), 0.5), orc.pattern_random(4, 1, len(ks), len(ns), 0.5),
                         orc.pattern_random(4, 2, len(ms), len(ns), 0.8)) if sparse else (None, None, None)
                for kind in (0, 1):
                    A = dbm.Matrix(ctx, 0, 0, 0, row_sizes=ms, col_sizes=ks, mask=masks[0])
                    B = dbm.Matrix(ctx, 0, 0, 0, row_sizes=ks, col_sizes=ns, mask=masks[1])
                    C = dbm.Matrix(ctx, 0, 0, 0, row_sizes=ms, col_sizes=ns, mask=masks[2])
                    A.fill_random(SEED, 0, kind)
                    B.fill_random(SEED, 1, kind)
                    with Watchdog(CASE_TIMEOUT):
                        for rep in range(2):  # second call: cached plan, the same exchange pool
                            C.fill_random(SEED, 2, kind)
                            dbm.multiply(ctx, 0.75, A, B, -1.25, C, path)
                        torch.cuda.synchronize()
                    got = C.arena.cpu().numpy()[: C.arena_bytes // 8]
                    Ad = orc.fill_dense(SEED, 0, kind, sum(ms), sum(ks))
                    Bd = orc.fill_dense(SEED, 1, kind, sum(ks), sum(ns))
                    Cd = orc.fill_dense(SEED, 2, kind, sum(ms), sum(ns))
                    ref = orc.nu_scatter(orc.nu_multiply(ms, ns, ks, 0.75, Ad, Bd, -1.25, Cd, *masks), ms, ns, pr, pc,
                                         r, c, masks[2])
                    if kind == 1:
                        ok = np.array_equal(got, ref)
                        err = float(np.abs(got - ref).max()) if ref.size else 0.0
                    else:
                        err = float(np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-300)) if ref.size else 0.0
                        ok = err <= 1e-12
                    flags = torch.tensor([0 if ok else 1], device=dev)
                    dist.all_reduce(flags)
                    ncases += 1
                    max_err = max(max_err, err)
                    failures += int(flags.item() > 0)
                    if rank == 0 or not ok:
                        print(json.dumps({"rank": rank, "grid": f"{pr}x{pc}", "nonuni": mi, "path": path,
                                          "sparse": sparse, "kind": kind, "err": err, "ok": bool(ok)}), flush=True)
        ctx.close()
    return failures, ncases, max_err


def sparse_recv_bytes(am, bm, bs, pr, pc, r, c):
    """Bytes rank (r, c) pulls in a block-sparse blocked multiply: the stored blocks of every remote
    A(r, kappa) / B(kappa, c) panel (owner-pull Cannon, reading R5; only stored blocks move, R15)."""
    L = orc.lcm(pr, pc)
    Mb, Kb = am.shape
    Nb = bm.shape[1]
    me = r * pc + c
    total = 0
    for s in range(L):
        k, asrc, bsrc = orc.cannon_step(pr, pc, r, c, s)
        if asrc != me:
            total += int(am[r:Mb:pr, k:Kb:L].sum())
        if bsrc != me:
            total += int(bm[k:Kb:L, c:Nb:pc].sum())
    return total * bs * bs * 8


def sparse_cases(world, rank, dev, grids):
    """Block-sparse operands (reading R15) on every grid: both paths against orc_multiply_sparse."""
    failures = ncases = 0
    max_err = 0.0
    shapes = [(352, 352, 352, 22, 0.3, 0.4, 1.0), (704, 528, 1100, 22, 0.1, 0.2, 0.7), (384, 640, 1280, 64, 0.5, 0.5, 0.5),
              (66, 154, 198, 22, 0.0, 0.5, 1.0)]
    for pr, pc in grids:
        ctx = dbm.Context.from_distributed(pr=pr, pc=pc)
        r, c = ctx.myrow, ctx.mycol
        for (M, N, K, bs, oa, ob, oc) in shapes:
            Mb, Nb, Kb = M // bs, N // bs, K // bs
            am, bm, cm = (orc.pattern_random(5, i, *dims, occ) for i, dims, occ in
                          ((0, (Mb, Kb), oa), (1, (Kb, Nb), ob), (2, (Mb, Nb), oc)))
            for path in ("blocked", "densified"):
                for kind in (0, 1):
                    A = dbm.Matrix(ctx, M, K, bs, mask=am)
                    B = dbm.Matrix(ctx, K, N, bs, mask=bm)
                    C = dbm.Matrix(ctx, M, N, bs, mask=cm)
                    A.fill_random(SEED, 0, kind)
                    B.fill_random(SEED, 1, kind)
                    with Watchdog(CASE_TIMEOUT):
                        for rep in range(2):
                            C.fill_random(SEED, 2, kind)
                            st = dbm.multiply(ctx, 0.75, A, B, -1.25, C, path)
                        torch.cuda.synchronize()
                    got = C.arena.cpu().numpy()[: C.arena_bytes // 8]
                    Ag = orc.fill_arena(SEED, 0, kind, M, K, bs)
                    Bg = orc.fill_arena(SEED, 1, kind, K, N, bs)
                    Cg = orc.fill_arena(SEED, 2, kind, M, N, bs)
                    orc.multiply_sparse(Mb, Nb, Kb, bs, 0.75, Ag, am, Bg, bm, -1.25, Cg, cm)
                    ref = orc.sparse_compress(Cg, cm, Mb, Nb, bs, pr, pc, r, c)
                    if kind == 1:
                        ok_val = np.array_equal(got, ref)
                        err = float(np.abs(got - ref).max()) if ref.size else 0.0
                    else:
                        err = float(np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-300)) if ref.size else 0.0
                        ok_val = err <= 1e-12
                    if path == "blocked":
                        ok_bytes = st["bytes_recv"] == sparse_recv_bytes(am, bm, bs, pr, pc, r, c)
                    else:
                        ok_bytes = (st["bytes_recv"], st["bytes_sent"]) == orc.cannon_bytes(Mb, Nb, Kb, bs, pr, pc, r, c)
                    flags = torch.tensor([0 if (ok_val and ok_bytes) else 1], device=dev)
                    dist.all_reduce(flags)
                    ncases += 1
                    max_err = max(max_err, err)
                    if flags.item():
                        failures += 1
                    if rank == 0 or not (ok_val and ok_bytes):
                        print(json.dumps({"rank": rank, "grid": f"{pr}x{pc}", "sparse": [oa, ob, oc],
                                          "shape": [M, N, K, bs], "path": path, "kind": kind, "err": err,
                                          "ok": bool(ok_val), "bytes_ok": ok_bytes, "recv": st["bytes_recv"]}),
                              flush=True)
        ctx.close()
    return failures, ncases, max_err


if __name__ == "__main__":
    main()
