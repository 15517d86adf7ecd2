"""CPU checks of the C ABI boundary: libdbm.so loads, exports every symbol include/dbm.h declares,
and its host-only schedule (dbm_plan_exchange) matches the oracle's Cannon plan.  No GPU calls."""
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "dbm.h")


@pytest.fixture(scope="module")
def dbm():
    from paper_1910_04796_b200 import build as b

    b.build()
    import paper_1910_04796_b200 as d

    d.load()
    return d


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dbm_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_exported(dbm):
    syms = declared_symbols()
    assert len(syms) >= 25
    out = subprocess.run(["nm", "-D", "--defined-only", dbm.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (dbm_\w+)", out))
    missing = [s for s in syms if s not in exported]
    assert not missing, missing
    # the Python binding marshals every one of them, by the same names
    assert sorted(dbm.EXPORTS) == syms


def test_library_is_sm100a_and_has_dmma_and_tma(dbm):
    sass = subprocess.run(["cuobjdump", "-sass", dbm.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in subprocess.run(["cuobjdump", "-lelf", dbm.LIB_PATH], capture_output=True, text=True).stdout
    assert "DMMA.8x8x4" in sass  # FP64 tensor-core path (mma.sync f64)
    assert "UTMALDG.2D" in sass  # TMA tile loads


def test_status_strings(dbm):
    lib = dbm.load()
    assert lib.dbm_status_string(0) == b"DBM_OK"
    assert lib.dbm_status_string(2) == b"DBM_ERR_SHAPE"
    assert lib.dbm_status_string(21) == b"DBM_ERR_NCCL"
    assert lib.dbm_unique_id_bytes() == 128


def test_plan_exchange_errors(dbm):
    with pytest.raises(dbm.DbmError) as e:
        dbm.plan_exchange(2, 2, 0, 0, 4, 4, 4, 22, 7)
    assert e.value.name == "DBM_ERR_RANGE"
    with pytest.raises(dbm.DbmError):
        dbm.plan_exchange(2, 2, 2, 0, 4, 4, 4, 22, 0)


GRIDS = [(1, 2), (2, 1), (2, 2), (2, 4), (4, 2), (1, 4), (4, 1), (3, 2)]


@pytest.mark.parametrize("pr,pc", GRIDS)
@pytest.mark.parametrize("path", ["densified", "blocked"])
def test_plan_exchange_matches_oracle_schedule(dbm, orc, pr, pc, path):
    """The library's send/recv lists realise the oracle's owner-pull schedule: every recv has a matching
    send on the peer with the same kappa and size, and per-rank byte totals equal orc_cannon_bytes
    (blocked path: panels of whole blocks, exactly the oracle's count)."""
    L = orc.lcm(pr, pc)
    Mb, Nb, Kb, bs = 7, 5, 11, 4
    tot_recv = {}
    tot_sent = {}
    for s in range(L):
        ops = {}
        for r in range(pr):
            for c in range(pc):
                ops[r * pc + c] = dbm.plan_exchange(pr, pc, r, c, Mb, Nb, Kb, bs, s, path)
        for me, lst in ops.items():
            r, c = divmod(me, pc)
            k, asrc, bsrc = orc.cannon_step(pr, pc, r, c, s)
            recvs = [o for o in lst if not o["send"]]
            assert {(o["operand"], o["peer"]) for o in recvs} == \
                ({("A", asrc)} if asrc != me else set()) | ({("B", bsrc)} if bsrc != me else set())
            for o in lst:
                assert o["kappa"] == (k if not o["send"] else o["kappa"])
                mirror = [q for q in ops[o["peer"]] if q["peer"] == me and q["send"] != o["send"]
                          and q["operand"] == o["operand"]]
                assert len(mirror) == 1 and mirror[0]["bytes"] == o["bytes"] and mirror[0]["kappa"] == o["kappa"]
                key = tot_sent if o["send"] else tot_recv
                key[me] = key.get(me, 0) + o["bytes"]
            # at most one send per operand per step
            assert sum(1 for o in lst if o["send"] and o["operand"] == "A") <= 1
            assert sum(1 for o in lst if o["send"] and o["operand"] == "B") <= 1
    if path == "blocked":
        for r in range(pr):
            for c in range(pc):
                rv, sd = orc.cannon_bytes(Mb, Nb, Kb, bs, pr, pc, r, c)
                assert tot_recv.get(r * pc + c, 0) == rv
                assert tot_sent.get(r * pc + c, 0) == sd


@pytest.mark.parametrize("pr,pc", [(1, 2), (2, 2), (2, 4), (4, 2), (1, 4), (3, 2)])
def test_plan_tallskinny_matches_oracle(dbm, orc, pr, pc):
    for shape in [(22, 22, 301, 64), (7, 5, 40, 22), (3, 9, 17, 2)]:
        for r in range(pr):
            for c in range(pc):
                assert dbm.plan_tallskinny(pr, pc, r, c, *shape) == orc.ts_bytes(*shape[:3], shape[3], pr, pc, r, c)


def test_pattern_random_matches_oracle(dbm, orc):
    """Host-only dbm_pattern_random (reading R15) against the oracle's independent implementation."""
    for occ in (0.0, 0.01, 0.37, 1.0):
        for seed, mid, Mb, Nb in ((1910, 0, 31, 47), (7, 5, 1, 90), (3, 2, 64, 1)):
            assert np.array_equal(dbm.pattern_random(seed, mid, Mb, Nb, occ), orc.pattern_random(seed, mid, Mb, Nb, occ))
    with pytest.raises(dbm.DbmError):
        dbm.pattern_random(1, 0, 4, 4, 1.5)


def test_pattern_product_matches_numpy(dbm, orc):
    """Host-only symbolic product (fill-in workflow, R15) vs numpy's boolean matrix product."""
    a = orc.pattern_random(2, 0, 23, 31, 0.1)
    b = orc.pattern_random(2, 1, 31, 17, 0.15)
    c0 = orc.pattern_random(2, 2, 23, 17, 0.3)
    want = ((a.astype(np.int64) @ b.astype(np.int64)) > 0).astype(np.uint8)
    assert np.array_equal(dbm.pattern_product(a, b), want)
    assert np.array_equal(dbm.pattern_product(a, b, c0), want | c0)


@pytest.mark.parametrize("pr,pc", GRIDS + [(3, 3), (4, 4), (2, 3), (1, 8), (8, 1)])
def test_first_step_is_local_first(dbm, orc, pr, pc):
    """dbm_debug_first_step (the copy-engine transport's local-first order): every rank starts at a
    canonical step with the most local operands any step offers it (brute force over the oracle's schedule,
    orc_cannon_step); on the 2 x 2 and 2 x 4 grids no owner serves more than one first-step pull (the
    canonical order makes one rank of 2 x 2 pull both operands and another serve both pulls)."""
    L = orc.lcm(pr, pc)
    served = {}
    for q in range(pr * pc):
        r, c = divmod(q, pc)
        first = dbm.debug_first_step(pr, pc, q)
        assert 0 <= first < L

        def local(s):
            _, a, b = orc.cannon_step(pr, pc, r, c, s)
            return (a == q) + (b == q)

        assert local(first) == max(local(s) for s in range(L))
        _, a, b = orc.cannon_step(pr, pc, r, c, first)
        for src in (a, b):
            if src != q:
                served[src] = served.get(src, 0) + 1
    if (pr, pc) in ((2, 2), (2, 4)):
        assert max(served.values(), default=0) <= 1
    with pytest.raises(dbm.DbmError):
        dbm.debug_first_step(pr, pc, pr * pc)
