"""TEST INFRASTRUCTURE ONLY — ctypes view of the host oracle (oracle/dbm_oracle.c).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / ``--impl reference``
legs may import this package.  The product (paper_1910_04796_b200/) never imports it and
shares no code with it.  This module only marshals numpy arrays into the C functions;
all arithmetic lives in dbm_oracle.c, each function citing the PAPER.md passage it follows.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "dbm_oracle.c")
_LIB = os.path.join(_HERE, "libdbm_oracle.so")

_i64 = C.c_int64
_i32 = C.c_int32
_u64 = C.c_uint64
_dbl = C.c_double
_pd = C.POINTER(C.c_double)
_pi64 = C.POINTER(C.c_int64)
_pi32 = C.POINTER(C.c_int32)
_pint = C.POINTER(C.c_int)
_pu8 = C.POINTER(C.c_uint8)


def build(force: bool = False) -> str:
    """Compile the oracle (plain C, OpenMP) next to its source."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
        os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "dbm_oracle.h"))
    ):
        subprocess.check_call(
            ["gcc", "-O2", "-std=c11", "-fopenmp", "-fPIC", "-shared", "-ffp-contract=off",
             "-o", _LIB + ".tmp", _SRC, "-lm"]
        )
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        sig = {
            "orc_grid_dims": (None, [C.c_int, _pint, _pint]),
            "orc_local_count": (_i64, [_i64, C.c_int, C.c_int]),
            "orc_owner_rank": (C.c_int, [_i64, _i64, C.c_int, C.c_int]),
            "orc_lcm": (_i64, [_i64, _i64]),
            "orc_fill_value": (_dbl, [_u64, C.c_uint32, _i64, _i64, C.c_int]),
            "orc_fill_arena": (None, [_u64, C.c_uint32, C.c_int, _i64, _i64, C.c_int, C.c_int, C.c_int,
                                      C.c_int, C.c_int, _pd]),
            "orc_scatter": (None, [_pd, _i64, _i64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _pd]),
            "orc_gather": (None, [_pd, _i64, _i64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _pd]),
            "orc_arena_to_dense": (None, [_pd, _i64, _i64, C.c_int, _pd]),
            "orc_dense_to_arena": (None, [_pd, _i64, _i64, C.c_int, _pd]),
            "orc_multiply_blocked": (None, [_i64, _i64, _i64, C.c_int, _dbl, _pd, _pd, _dbl, _pd]),
            "orc_dense_gemm": (None, [_i64, _i64, _i64, _dbl, _pd, _pd, _dbl, _pd]),
            "orc_traversal": (_i64, [_i64, _i64, _pi64, _pi64]),
            "orc_stacks": (_i64, [_i64, _i64, _i64, _i64, _pi32, _pi64, _pi64]),
            "orc_cannon_step": (None, [C.c_int] * 5 + [_pint, _pint, _pint]),
            "orc_cannon_bytes": (None, [_i64, _i64, _i64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                        _pi64, _pi64]),
            "orc_densified_dims": (None, [_i64] * 5 + [_pi64] * 4),
            "orc_ts_bytes": (None, [_i64, _i64, _i64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _pi64, _pi64]),
            "orc_densify_cols": (None, [_pd, _i64, _i64, C.c_int, _pi64, _i64, _pd, _i64, C.c_int]),
            "orc_densify_rows": (None, [_pd, _i64, _i64, C.c_int, _pi64, _i64, _pd, _i64, C.c_int]),
            "orc_pack_panel": (None, [_pd, _i64, _i64, C.c_int, C.c_int, _pi64, _i64, _pd]),
            "orc_undensify": (None, [_pd, _i64, _i64, _i64, C.c_int, _dbl, _dbl, _pd]),
            "orc_rows_from_seeds": (None, [_i64, _i64, _i64, _u64, C.c_int, _dbl, _dbl, _pi64, _i64, _pd]),
            "orc_freivalds_rhs": (None, [_i64, _i64, _i64, _u64, C.c_int, _dbl, _dbl, _u64, _pd, _pd]),
            "orc_sign_value": (_dbl, [_u64, _i64]),
            "orc_num_threads": (C.c_int, []),
            "orc_nu_local_elems": (_i64, [_pi32, _i64, _pi32, _i64, C.c_int, C.c_int, C.c_int, C.c_int, _pu8]),
            "orc_nu_scatter": (None, [_pd, _pi32, _i64, _pi32, _i64, C.c_int, C.c_int, C.c_int, C.c_int, _pu8, _pd]),
            "orc_nu_gather": (None, [_pd, _pi32, _i64, _pi32, _i64, C.c_int, C.c_int, C.c_int, C.c_int, _pu8, _pd]),
            "orc_nu_multiply": (None, [_pi32, _i64, _pi32, _i64, _pi32, _i64, _dbl, _pd, _pu8, _pd, _pu8, _dbl, _pd,
                                       _pu8]),
            "orc_pattern_present": (C.c_int, [_u64, C.c_uint32, _i64, _i64, _dbl]),
            "orc_pattern_random": (None, [_u64, C.c_uint32, _i64, _i64, _dbl, _pu8]),
            "orc_multiply_sparse": (None, [_i64, _i64, _i64, C.c_int, _dbl, _pd, _pu8, _pd, _pu8, _dbl, _pd, _pu8]),
            "orc_sparse_compress": (_i64, [_pd, _pu8, _i64, _i64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                           _pd]),
            "orc_sparse_expand": (None, [_pd, _pu8, _i64, _i64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _pd]),
            "orc_sparse_stacks": (_i64, [_i64, _i64, _i64, _pu8, _pu8, _pu8, _i64, _pi32, _pi64, _pi64]),
            "orc_sparse_rows_from_seeds": (_i64, [_i64, _i64, _i64, C.c_int, _u64, C.c_int, _u64, _dbl, _dbl, _dbl,
                                                  _dbl, _dbl, _pi64, _i64, _pd]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _p(a: np.ndarray, ct=_pd):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ct)


# ---------------------------------------------------------------- distribution
def grid_dims(nranks: int) -> tuple[int, int]:
    pr, pc = C.c_int(), C.c_int()
    lib().orc_grid_dims(nranks, C.byref(pr), C.byref(pc))
    return pr.value, pc.value


def local_count(nblocks: int, p: int, r: int) -> int:
    return lib().orc_local_count(nblocks, p, r)


def owner_rank(bi: int, bj: int, pr: int, pc: int) -> int:
    return lib().orc_owner_rank(bi, bj, pr, pc)


def lcm(a: int, b: int) -> int:
    return lib().orc_lcm(a, b)


# ---------------------------------------------------------------- input generator
def fill_value(seed: int, mat_id: int, gi: int, gj: int, kind: int = 0) -> float:
    return lib().orc_fill_value(seed, mat_id, gi, gj, kind)


def fill_arena(seed, mat_id, kind, rows, cols, bs, pr=1, pc=1, r=0, c=0) -> np.ndarray:
    mloc = local_count(rows // bs, pr, r)
    nloc = local_count(cols // bs, pc, c)
    a = np.empty(mloc * nloc * bs * bs, dtype=np.float64)
    lib().orc_fill_arena(seed, mat_id, kind, rows, cols, bs, pr, pc, r, c, _p(a))
    return a


def scatter(g, Mb, Nb, bs, pr, pc, r, c) -> np.ndarray:
    out = np.empty(local_count(Mb, pr, r) * local_count(Nb, pc, c) * bs * bs)
    lib().orc_scatter(_p(g), Mb, Nb, bs, pr, pc, r, c, _p(out))
    return out


def gather_into(g, local, Mb, Nb, bs, pr, pc, r, c) -> None:
    lib().orc_gather(_p(local), Mb, Nb, bs, pr, pc, r, c, _p(g))


def arena_to_dense(g, Mb, Nb, bs) -> np.ndarray:
    """Returns the dense matrix as a (rows, cols) numpy array (column-major storage)."""
    d = np.empty(Mb * bs * Nb * bs)
    lib().orc_arena_to_dense(_p(g), Mb, Nb, bs, _p(d))
    return d.reshape(Nb * bs, Mb * bs).T


def dense_to_arena(d: np.ndarray, bs: int) -> np.ndarray:
    M, N = d.shape
    dc = np.ascontiguousarray(d.T)  # column-major storage
    g = np.empty(M * N)
    lib().orc_dense_to_arena(_p(dc), M // bs, N // bs, bs, _p(g))
    return g


# ---------------------------------------------------------------- product
def multiply_blocked(Mb, Nb, Kb, bs, alpha, A, B, beta, C) -> None:
    lib().orc_multiply_blocked(Mb, Nb, Kb, bs, alpha, _p(A), _p(B), beta, _p(C))


def dense_gemm(alpha, A: np.ndarray, B: np.ndarray, beta, Cm: np.ndarray) -> np.ndarray:
    M, K = A.shape
    N = B.shape[1]
    a = np.ascontiguousarray(A.T)
    b = np.ascontiguousarray(B.T)
    c = np.ascontiguousarray(Cm.T)
    lib().orc_dense_gemm(M, N, K, alpha, _p(a), _p(b), beta, _p(c))
    return c.T


# ---------------------------------------------------------------- traversal / stacks
def traversal(mloc: int, nloc: int) -> np.ndarray:
    li = np.empty(max(mloc * nloc, 1), dtype=np.int64)
    lj = np.empty_like(li)
    n = lib().orc_traversal(mloc, nloc, _p(li, _pi64), _p(lj, _pi64))
    return np.stack([li[:n], lj[:n]], axis=1)


def stacks(mloc: int, nloc: int, kb: int, cap: int = 30000, counts_only: bool = False):
    ns = C.c_int64()
    if counts_only:
        e = lib().orc_stacks(mloc, nloc, kb, cap, None, None, C.byref(ns))
        return e, ns.value
    n = mloc * nloc * kb
    trip = np.empty(max(3 * n, 3), dtype=np.int32)
    ptr = np.empty(n + 2, dtype=np.int64)
    e = lib().orc_stacks(mloc, nloc, kb, cap, _p(trip, _pi32), _p(ptr, _pi64), C.byref(ns))
    return trip[: 3 * e].reshape(e, 3), ptr[: ns.value + 1]


# ---------------------------------------------------------------- block sparsity (reading R15)
def pattern_present(seed, mat_id, bi, bj, occupancy) -> bool:
    return bool(lib().orc_pattern_present(seed, mat_id, bi, bj, occupancy))


def pattern_random(seed, mat_id, Mb, Nb, occupancy) -> np.ndarray:
    """(Mb, Nb) uint8 mask of stored blocks."""
    m = np.empty(max(Mb * Nb, 1), dtype=np.uint8)
    lib().orc_pattern_random(seed, mat_id, Mb, Nb, occupancy, _p(m, _pu8))
    return m[: Mb * Nb].reshape(Mb, Nb)


def multiply_sparse(Mb, Nb, Kb, bs, alpha, A, amask, B, bmask, beta, Cg, cmask) -> None:
    am, bm, cm = (np.ascontiguousarray(x, dtype=np.uint8) for x in (amask, bmask, cmask))
    lib().orc_multiply_sparse(Mb, Nb, Kb, bs, alpha, _p(A), _p(am, _pu8), _p(B), _p(bm, _pu8), beta, _p(Cg),
                              _p(cm, _pu8))


def sparse_compress(g, mask, Mb, Nb, bs, pr=1, pc=1, r=0, c=0) -> np.ndarray:
    m = np.ascontiguousarray(mask, dtype=np.uint8)
    n = lib().orc_sparse_compress(_p(g), _p(m, _pu8), Mb, Nb, bs, pr, pc, r, c, None)
    out = np.empty(max(n * bs * bs, 1))
    lib().orc_sparse_compress(_p(g), _p(m, _pu8), Mb, Nb, bs, pr, pc, r, c, _p(out))
    return out[: n * bs * bs]


def sparse_expand_into(g, local, mask, Mb, Nb, bs, pr=1, pc=1, r=0, c=0) -> None:
    m = np.ascontiguousarray(mask, dtype=np.uint8)
    loc = np.ascontiguousarray(local, dtype=np.float64)
    if loc.size == 0:
        loc = np.zeros(1)
    lib().orc_sparse_expand(_p(loc), _p(m, _pu8), Mb, Nb, bs, pr, pc, r, c, _p(g))


def sparse_stacks(amask, bmask, cmask, cap: int = 30000):
    """amask (mloc, kb), bmask (kb, nloc), cmask (mloc, nloc) -> (triplets (E,3) int32, stack_ptr)."""
    am, bm, cm = (np.ascontiguousarray(x, dtype=np.uint8) for x in (amask, bmask, cmask))
    mloc, kb = am.shape
    nloc = bm.shape[1]
    ns = C.c_int64()
    e = lib().orc_sparse_stacks(mloc, nloc, kb, _p(am, _pu8), _p(bm, _pu8), _p(cm, _pu8), cap, None, None,
                                C.byref(ns))
    trip = np.empty(max(3 * e, 3), dtype=np.int32)
    ptr = np.empty(ns.value + 2, dtype=np.int64)
    lib().orc_sparse_stacks(mloc, nloc, kb, _p(am, _pu8), _p(bm, _pu8), _p(cm, _pu8), cap, _p(trip, _pi32),
                            _p(ptr, _pi64), C.byref(ns))
    return trip[: 3 * e].reshape(e, 3), ptr[: ns.value + 1]


def sparse_rows_from_seeds(M, N, K, bs, seed, kind, pseed, occ_a, occ_b, occ_c, alpha, beta, rows):
    """(out (nrows, N) with NaN on absent C blocks, multiply-adds performed)."""
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    out = np.empty((len(rows), N))
    n = lib().orc_sparse_rows_from_seeds(M, N, K, bs, seed, kind, pseed, occ_a, occ_b, occ_c, alpha, beta,
                                         _p(rows, _pi64), len(rows), _p(out))
    return out, n


# ---------------------------------------------------------------- Cannon
def cannon_step(pr, pc, r, c, s) -> tuple[int, int, int]:
    k, a, b = C.c_int(), C.c_int(), C.c_int()
    lib().orc_cannon_step(pr, pc, r, c, s, C.byref(k), C.byref(a), C.byref(b))
    return k.value, a.value, b.value


def cannon_bytes(Mb, Nb, Kb, bs, pr, pc, r, c) -> tuple[int, int]:
    rv, sd = C.c_int64(), C.c_int64()
    lib().orc_cannon_bytes(Mb, Nb, Kb, bs, pr, pc, r, c, C.byref(rv), C.byref(sd))
    return rv.value, sd.value


def ts_bytes(Mb, Nb, Kb, bs, pr, pc, r, c) -> tuple[int, int]:
    rv, sd = C.c_int64(), C.c_int64()
    lib().orc_ts_bytes(Mb, Nb, Kb, bs, pr, pc, r, c, C.byref(rv), C.byref(sd))
    return rv.value, sd.value


# ---------------------------------------------------------------- densify
def densified_dims(M, N, K, pt, t):
    v = [C.c_int64() for _ in range(4)]
    lib().orc_densified_dims(M, N, K, pt, t, *[C.byref(x) for x in v])
    return (v[0].value, v[1].value), (v[2].value, v[3].value)


def densify_cols(arena, mloc, nloc, bs, kcols, layout=0) -> np.ndarray:
    kc = np.ascontiguousarray(kcols, dtype=np.int64)
    nk = len(kc)
    if layout == 0:
        ld = mloc * bs
        d = np.zeros(ld * nk * bs)
    else:
        ld = nk * bs
        d = np.zeros(mloc * bs * ld)
    lib().orc_densify_cols(_p(arena), mloc, nloc, bs, _p(kc, _pi64), nk, _p(d), ld, layout)
    return d


def densify_rows(arena, mloc, nloc, bs, krows, layout=0) -> np.ndarray:
    kr = np.ascontiguousarray(krows, dtype=np.int64)
    nk = len(kr)
    if layout == 0:
        ld = nk * bs
        d = np.zeros(ld * nloc * bs)
    else:
        ld = nloc * bs
        d = np.zeros(nk * bs * ld)
    lib().orc_densify_rows(_p(arena), mloc, nloc, bs, _p(kr, _pi64), nk, _p(d), ld, layout)
    return d


def pack_panel(arena, mloc, nloc, bs, operand, kidx) -> np.ndarray:
    """Packed Cannon panel of whole blocks (a3): A (operand 0) blocks (li, kidx[q]) row-major over (li, q);
    B (operand 1) blocks (kidx[q], lj) row-major over (q, lj)."""
    k = np.ascontiguousarray(kidx, dtype=np.int64)
    n = (mloc if operand == 0 else nloc) * len(k) * bs * bs
    out = np.zeros(max(n, 1))
    lib().orc_pack_panel(_p(arena), mloc, nloc, bs, operand, _p(k, _pi64), len(k), _p(out))
    return out[:n]


def undensify(dense, ld, mloc, nloc, bs, alpha, beta, arena) -> None:
    lib().orc_undensify(_p(dense), ld, mloc, nloc, bs, alpha, beta, _p(arena))


# ---------------------------------------------------------------- verification from seeds
def rows_from_seeds(M, N, K, seed, kind, alpha, beta, rows) -> np.ndarray:
    r = np.ascontiguousarray(rows, dtype=np.int64)
    out = np.empty(len(r) * N)
    lib().orc_rows_from_seeds(M, N, K, seed, kind, alpha, beta, _p(r, _pi64), len(r), _p(out))
    return out.reshape(len(r), N)


def freivalds_rhs(M, N, K, seed, kind, alpha, beta, x_seed):
    x = np.empty(N)
    out = np.empty(M)
    lib().orc_freivalds_rhs(M, N, K, seed, kind, alpha, beta, x_seed, _p(x), _p(out))
    return x, out


def num_threads() -> int:
    return lib().orc_num_threads()


# ---------------------------------------------------------------- non-uniform block sizes (reading R16)
def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def _mask(m):
    return None if m is None else np.ascontiguousarray(m, dtype=np.uint8)


def fill_dense(seed, mat_id, kind, rows, cols) -> np.ndarray:
    """The generator's matrix as a dense column-major (rows, cols) array: D(gi, gj) = v(seed, mat_id, gi, gj)
    (independent of any blocking, so it is the reference for every block-size layout)."""
    d = np.empty((cols, rows))
    for gj in range(cols):
        for gi in range(rows):
            d[gj, gi] = fill_value(seed, mat_id, gi, gj, kind)
    return d.T  # (rows, cols) view of column-major storage


def nu_local_elems(rsz, csz, pr=1, pc=1, r=0, c=0, mask=None) -> int:
    rs, cs = _i32(rsz), _i32(csz)
    mk = _mask(mask)
    return lib().orc_nu_local_elems(_p(rs, _pi32), len(rs), _p(cs, _pi32), len(cs), pr, pc, r, c,
                                    _p(mk, _pu8) if mk is not None else None)


def nu_scatter(dense, rsz, csz, pr=1, pc=1, r=0, c=0, mask=None) -> np.ndarray:
    """Local arena of rank (r, c) from a dense (rows, cols) array (any memory order)."""
    rs, cs = _i32(rsz), _i32(csz)
    mk = _mask(mask)
    d = np.ascontiguousarray(np.asarray(dense).T)  # column-major storage
    out = np.empty(max(nu_local_elems(rs, cs, pr, pc, r, c, mk), 1))
    lib().orc_nu_scatter(_p(d), _p(rs, _pi32), len(rs), _p(cs, _pi32), len(cs), pr, pc, r, c,
                         _p(mk, _pu8) if mk is not None else None, _p(out))
    return out[: nu_local_elems(rs, cs, pr, pc, r, c, mk)]


def nu_gather_into(dense_t, local, rsz, csz, pr=1, pc=1, r=0, c=0, mask=None) -> None:
    """Write rank (r, c)'s blocks into dense_t, a C-contiguous (cols, rows) array = column-major storage."""
    rs, cs = _i32(rsz), _i32(csz)
    mk = _mask(mask)
    lib().orc_nu_gather(_p(np.ascontiguousarray(local)), _p(rs, _pi32), len(rs), _p(cs, _pi32), len(cs), pr, pc, r,
                        c, _p(mk, _pu8) if mk is not None else None, _p(dense_t))


def nu_multiply(msz, nsz, ksz, alpha, A, B, beta, C, amask=None, bmask=None, cmask=None) -> np.ndarray:
    """C_out (dense (M, N)) = alpha*A*B + beta*C over stored blocks of mixed (m, n, k) sizes."""
    ms, ns, ks = _i32(msz), _i32(nsz), _i32(ksz)
    a = np.ascontiguousarray(np.asarray(A).T)
    b = np.ascontiguousarray(np.asarray(B).T)
    cc = np.ascontiguousarray(np.asarray(C).T).copy()
    am, bm, cm = _mask(amask), _mask(bmask), _mask(cmask)
    lib().orc_nu_multiply(_p(ms, _pi32), len(ms), _p(ns, _pi32), len(ns), _p(ks, _pi32), len(ks), alpha, _p(a),
                          _p(am, _pu8) if am is not None else None, _p(b), _p(bm, _pu8) if bm is not None else None,
                          beta, _p(cc), _p(cm, _pu8) if cm is not None else None)
    return cc.T
