"""Multi-process (world_size 2, 4 and 8, gloo, CPU) test of the library's Cannon exchange schedule.

Each rank asks libdbm (host-only dbm_plan_exchange, the same op list dbm_multiply hands to NCCL)
what to send and receive at every step, moves real panels with torch.distributed send/recv over
gloo, multiplies them with numpy, and the gathered C must equal the oracle's product.  This covers
the N>1 host logic without a GPU (reading R5 owner-pull schedule)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, pr, pc, port, shape, q):
    import sys

    sys.path.insert(0, ROOT)
    import oracle as orc
    import paper_1910_04796_b200 as dbm

    try:
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        Mb, Nb, Kb, bs = shape
        r, c = divmod(rank, pc)
        L = orc.lcm(pr, pc)
        seed = 1910
        Aloc = orc.fill_arena(seed, 0, 0, Mb * bs, Kb * bs, bs, pr, pc, r, c)
        Bloc = orc.fill_arena(seed, 1, 0, Kb * bs, Nb * bs, bs, pr, pc, r, c)
        mloc, nloc = orc.local_count(Mb, pr, r), orc.local_count(Nb, pc, c)
        kA, kB = orc.local_count(Kb, pc, c), orc.local_count(Kb, pr, r)

        def a_panel(k):  # dense (mloc*bs) x (kb*bs) of my A blocks with global k' = k mod L
            cols = [kl for kl in range(kA) if (c + kl * pc) % L == k]
            d = orc.densify_cols(Aloc, mloc, kA, bs, cols, 1) if mloc and cols else np.zeros(0)
            return d.reshape(mloc * bs, len(cols) * bs)

        def b_panel(k):
            rows = [kl for kl in range(kB) if (r + kl * pr) % L == k]
            d = orc.densify_rows(Bloc, kB, nloc, bs, rows, 1) if nloc and rows else np.zeros(0)
            return d.reshape(len(rows) * bs, nloc * bs)

        Cloc = np.zeros((mloc * bs, nloc * bs))
        for s in range(L):
            ops = dbm.plan_exchange(pr, pc, r, c, Mb, Nb, Kb, bs, s, "blocked")
            k_me, asrc, bsrc = orc.cannon_step(pr, pc, r, c, s)
            reqs, recv = [], {}
            for o in ops:
                if o["send"]:
                    pan = a_panel(o["kappa"]) if o["operand"] == "A" else b_panel(o["kappa"])
                    assert pan.nbytes == o["bytes"]
                    reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(pan)), o["peer"]))
                else:
                    kbk = orc.local_count(Kb, L, o["kappa"])
                    shp = (mloc * bs, kbk * bs) if o["operand"] == "A" else (kbk * bs, nloc * bs)
                    buf = torch.empty(shp, dtype=torch.float64)
                    assert buf.numel() * 8 == o["bytes"]
                    reqs.append(dist.irecv(buf, o["peer"]))
                    recv[o["operand"]] = buf
            for rq in reqs:
                rq.wait()
            Ap = recv["A"].numpy() if "A" in recv else a_panel(k_me)
            Bp = recv["B"].numpy() if "B" in recv else b_panel(k_me)
            assert ("A" in recv) == (asrc != rank) and ("B" in recv) == (bsrc != rank)
            if Ap.size and Bp.size:
                Cloc += Ap @ Bp
        # compare my share with the oracle's product
        A = orc.fill_arena(seed, 0, 0, Mb * bs, Kb * bs, bs)
        B = orc.fill_arena(seed, 1, 0, Kb * bs, Nb * bs, bs)
        Cg = np.zeros(Mb * Nb * bs * bs)
        orc.multiply_blocked(Mb, Nb, Kb, bs, 1.0, A, B, 0.0, Cg)
        ref = orc.scatter(Cg, Mb, Nb, bs, pr, pc, r, c)
        mine = np.zeros(mloc * nloc * bs * bs)
        if mloc and nloc:
            orc.dense_to_arena  # noqa: B018  (layout helper below)
            for li in range(mloc):
                for lj in range(nloc):
                    blk = Cloc[li * bs:(li + 1) * bs, lj * bs:(lj + 1) * bs]
                    mine[(li * nloc + lj) * bs * bs:(li * nloc + lj + 1) * bs * bs] = blk.T.reshape(-1)
        err = np.abs(mine - ref).max() if ref.size else 0.0
        q.put((rank, float(err)))
        dist.destroy_process_group()
    except Exception as e:  # surface to the parent
        q.put((rank, repr(e)))


@pytest.mark.parametrize("pr,pc,shape", [(1, 2, (3, 5, 7, 4)), (2, 1, (5, 3, 4, 2)), (2, 2, (5, 7, 9, 2)),
                                         (1, 4, (3, 9, 10, 2)), (4, 1, (9, 2, 5, 2)),
                                         # world 8: the north star's 2 x 4 grid (L = 4) and its transpose,
                                         # ragged block counts (13 = 4 + 3 + 3 + 3 K-blocks per panel)
                                         (2, 4, (5, 11, 13, 2)), (4, 2, (9, 5, 11, 3))])
def test_gloo_cannon_exchange(pr, pc, shape):
    world = pr * pc
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, pr, pc, port, shape, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, err in res:
        assert not isinstance(err, str), f"rank {rank}: {err}"
        assert err < 1e-12, (rank, err)
