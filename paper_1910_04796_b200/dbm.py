"""Thin Python binding of libdbm (include/dbm.h): argument marshalling only.

Every step of the multiply runs in the CUDA kernels of libdbm.so; PyTorch provides device memory
(tensors as arenas and workspace), the stream, and torch.distributed for the NCCL id broadcast.
There is no fallback: if libdbm.so is missing or a CUDA device is absent, the calls raise.
Names follow include/dbm.h (dbm_multiply -> multiply, dbm_matrix_fill_random -> Matrix.fill_random ...).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libdbm.so")

PATH_BLOCKED = 0
PATH_DENSIFIED = 1
PATH_AUTO = 2
_PATHS = {"blocked": PATH_BLOCKED, "densified": PATH_DENSIFIED, "auto": PATH_AUTO, PATH_BLOCKED: 0,
          PATH_DENSIFIED: 1, PATH_AUTO: 2}

# dbm_ctx_profile_read kernel ids
K_DGEMM, K_SMM, K_DENSIFY, K_UNDENSIFY, K_STACKGEN, K_EXCHANGE = 0, 1, 2, 3, 4, 5


class DbmError(RuntimeError):
    def __init__(self, status: int, name: str, detail: str):
        super().__init__(f"{name}: {detail}")
        self.status = status
        self.name = name


class Stats(C.Structure):
    _fields_ = [("entries", C.c_int64), ("stacks", C.c_int64), ("bytes_sent", C.c_int64),
                ("bytes_recv", C.c_int64), ("steps", C.c_int64), ("gemm_launches", C.c_int64),
                ("kernel_launches", C.c_int64), ("flops", C.c_double), ("ms_total", C.c_double),
                ("ms_densify", C.c_double), ("ms_local", C.c_double), ("ms_comm_exposed", C.c_double),
                ("ms_undensify", C.c_double)]

    def as_dict(self) -> dict:
        return {f: getattr(self, f) for f, _ in self._fields_}


_lib = None

_P = C.c_void_p
_I64 = C.c_int64
_SIGS = {
    "dbm_status_string": (C.c_char_p, [C.c_int]),
    "dbm_last_error": (C.c_char_p, []),
    "dbm_unique_id_bytes": (C.c_int, []),
    "dbm_get_unique_id": (C.c_int, [_P]),
    "dbm_ctx_create": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, _P, C.c_int, _P, C.POINTER(_P)]),
    "dbm_ctx_grid": (C.c_int, [_P] + [C.POINTER(C.c_int)] * 4),
    "dbm_ctx_set_stream": (C.c_int, [_P, _P]),
    "dbm_ctx_sync": (C.c_int, [_P]),
    "dbm_ctx_set_profiling": (C.c_int, [_P, C.c_int]),
    "dbm_ctx_profile_read": (C.c_int, [_P, C.c_int, C.POINTER(C.c_double), C.POINTER(_I64),
                                       C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "dbm_multiply_timing": (C.c_int, [_P, C.POINTER(Stats)]),
    "dbm_ctx_profile_timeline": (C.c_int, [_P, C.c_int, _P, C.POINTER(C.c_int)]),
    "dbm_ctx_launch_count": (C.c_int, [_P, C.POINTER(_I64)]),
    "dbm_ctx_set_dense_chunk_bytes": (C.c_int, [_P, _I64]),
    "dbm_ctx_set_transport": (C.c_int, [_P, C.c_int]),
    "dbm_ctx_set_algorithm": (C.c_int, [_P, C.c_int]),
    "dbm_plan_tallskinny": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, _I64, _I64, _I64, C.c_int32,
                                      C.POINTER(_I64), C.POINTER(_I64)]),
    "dbm_debug_first_step": (C.c_int, [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int)]),
    "dbm_plan_exchange": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, _I64, _I64, _I64, C.c_int32, C.c_int,
                                    C.c_int, _P, _P, C.POINTER(C.c_int)]),
    "dbm_ctx_destroy": (C.c_int, [_P]),
    "dbm_matrix_create": (C.c_int, [_P, _I64, _I64, C.c_int32, C.POINTER(_P)]),
    "dbm_matrix_create_sparse": (C.c_int, [_P, _I64, _I64, C.c_int32, _P, C.POINTER(_P)]),
    "dbm_pattern_random": (C.c_int, [C.c_uint64, C.c_uint32, _I64, _I64, C.c_double, _P]),
    "dbm_matrix_create_blocked": (C.c_int, [_P, _I64, _P, _I64, _P, _P, C.POINTER(_P)]),
    "dbm_matrix_block_sizes": (C.c_int, [_P, _P, _P]),
    "dbm_matrix_nnz": (C.c_int, [_P, C.POINTER(_I64), C.POINTER(_I64)]),
    "dbm_pattern_product": (C.c_int, [_I64, _I64, _I64, _P, _P, _P]),
    "dbm_ctx_set_densify_threshold": (C.c_int, [_P, C.c_double]),
    "dbm_matrix_local_info": (C.c_int, [_P, C.POINTER(_I64), C.POINTER(_I64), C.POINTER(_I64)]),
    "dbm_matrix_local_csr": (C.c_int, [_P, _P, _P, _P]),
    "dbm_matrix_attach": (C.c_int, [_P, _P, _I64]),
    "dbm_matrix_fill_random": (C.c_int, [_P, C.c_uint64, C.c_uint32, C.c_int]),
    "dbm_matrix_set_block": (C.c_int, [_P, _I64, _I64, _P]),
    "dbm_matrix_get_block": (C.c_int, [_P, _I64, _I64, _P]),
    "dbm_matrix_upload": (C.c_int, [_P, _P]),
    "dbm_matrix_download": (C.c_int, [_P, _P]),
    "dbm_owner_of_block": (C.c_int, [_P, _I64, _I64, C.POINTER(C.c_int)]),
    "dbm_matrix_destroy": (C.c_int, [_P]),
    "dbm_multiply_workspace": (C.c_int, [_P, _P, _P, _P, C.c_int, C.POINTER(_I64)]),
    "dbm_multiply": (C.c_int, [_P, C.c_double, _P, _P, C.c_double, _P, C.c_int, C.c_int32, _P, _I64,
                               C.POINTER(Stats)]),
    "dbm_multiply_host": (C.c_int, [_P, C.c_double, _P, _P, C.c_double, _P, C.c_int, C.c_int32, _P, _I64, _P, _P,
                                    _P, C.POINTER(Stats)]),
    "dbm_densify": (C.c_int, [_P, _P, _I64, C.c_int]),
    "dbm_undensify": (C.c_int, [_P, _P, _I64, C.c_double, C.c_double]),
    "dbm_debug_stacks": (C.c_int, [_P, _P, _P, _P, C.c_int, C.c_int32, _P, C.POINTER(_I64), _P,
                                   C.POINTER(_I64)]),
    "dbm_debug_pack_panel": (C.c_int, [_P, C.c_int, _I64, _I64, _I64, _I64, _P]),
    "dbm_debug_dgemm": (C.c_int, [_P, _I64, _I64, _I64, C.c_double, _P, _I64, _P, _I64, C.c_double, _P, _I64,
                                  C.c_int, _P, _I64]),
}
EXPORTS = tuple(_SIGS)


def load(path: str = LIB_PATH):
    """Load libdbm.so (no fallback: raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(path):
            raise RuntimeError(f"{path} is missing: run `python -m paper_1910_04796_b200.build` "
                               "(there is no CPU fallback)")
        lib = C.CDLL(path)
        for name, (res, args) in _SIGS.items():
            f = getattr(lib, name)
            f.restype = res
            f.argtypes = args
        _lib = lib
    return _lib


def _check(status: int) -> None:
    if status != 0:
        lib = load()
        raise DbmError(status, lib.dbm_status_string(status).decode(), lib.dbm_last_error().decode())


def _stream_ptr(stream) -> int | None:
    if stream is None:
        return None
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


# ---------------------------------------------------------------------------- context
class Context:
    """dbm_ctx: one rank's view of the Pr x Pc process grid (§II), one rank per GPU."""

    def __init__(self, nranks: int = 1, rank: int = 0, device: int | None = None, pr: int = 0, pc: int = 0,
                 unique_id: bytes | None = None, stream=None):
        lib = load()
        if device is None:
            device = torch.cuda.current_device()
        self.device = torch.device("cuda", device)
        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        self.stream = stream
        h = C.c_void_p()
        idbuf = C.create_string_buffer(unique_id, len(unique_id)) if unique_id else None
        _check(lib.dbm_ctx_create(nranks, rank, pr, pc, idbuf, device, _stream_ptr(stream), C.byref(h)))
        self.h = h
        self.nranks, self.rank = nranks, rank
        a = [C.c_int() for _ in range(4)]
        _check(lib.dbm_ctx_grid(h, *[C.byref(x) for x in a]))
        self.pr, self.pc, self.myrow, self.mycol = (x.value for x in a)
        self._ws = None

    @classmethod
    def from_distributed(cls, stream=None, pr: int = 0, pc: int = 0) -> "Context":
        """Build a context over torch.distributed's world (NCCL id broadcast from rank 0)."""
        import torch.distributed as dist

        world, rank = dist.get_world_size(), dist.get_rank()
        local = int(os.environ.get("LOCAL_RANK", rank % max(torch.cuda.device_count(), 1)))
        uid = None
        if world > 1:
            lib = load()
            obj = [None]
            if rank == 0:
                buf = C.create_string_buffer(lib.dbm_unique_id_bytes())
                _check(lib.dbm_get_unique_id(buf))
                obj[0] = buf.raw
            dist.broadcast_object_list(obj, src=0)
            uid = obj[0]
        return cls(world, rank, device=local, pr=pr, pc=pc, unique_id=uid, stream=stream)

    def set_stream(self, stream) -> None:
        self.stream = stream
        _check(load().dbm_ctx_set_stream(self.h, _stream_ptr(stream)))

    def sync(self) -> None:
        _check(load().dbm_ctx_sync(self.h))

    def set_profiling(self, on: bool) -> None:
        _check(load().dbm_ctx_set_profiling(self.h, int(on)))

    def profile_read(self, kernel: int) -> dict:
        ms, fl, by = C.c_double(), C.c_double(), C.c_double()
        n = C.c_int64()
        _check(load().dbm_ctx_profile_read(self.h, kernel, C.byref(ms), C.byref(n), C.byref(fl), C.byref(by)))
        return {"ms": ms.value, "launches": n.value, "flops": fl.value, "bytes": by.value}

    def multiply_timing(self) -> dict:
        """dbm_multiply_timing: ms_total / ms_densify / ms_local / ms_comm_exposed / ms_undensify of the last
        multiply run with profiling on."""
        st = Stats()
        _check(load().dbm_multiply_timing(self.h, C.byref(st)))
        return {k: getattr(st, k) for k in ("ms_total", "ms_densify", "ms_local", "ms_comm_exposed", "ms_undensify")}

    def profile_timeline(self, max_records: int = 4096) -> list[tuple[int, float, float]]:
        """dbm_ctx_profile_timeline: (kind, start_ms, end_ms) of the pending profiling records."""
        import numpy as np

        buf = np.zeros(3 * max(max_records, 1))
        n = C.c_int()
        _check(load().dbm_ctx_profile_timeline(self.h, max_records, buf.ctypes.data, C.byref(n)))
        k = min(n.value, max_records)
        return [(int(buf[3 * i]), float(buf[3 * i + 1]), float(buf[3 * i + 2])) for i in range(k)]

    def set_transport(self, transport: str | int) -> None:
        """'ce' (copy engines over CUDA IPC, default) or 'nccl' (grouped send/recv)."""
        t = {"ce": 0, "nccl": 1}.get(transport, transport)
        _check(load().dbm_ctx_set_transport(self.h, int(t)))
        self.transport = t

    def set_algorithm(self, algorithm: str | int) -> None:
        """'cannon' (default), 'tallskinny' (densified path, copy-engine transport) or 'auto'
        (tall-and-skinny when K >= 16 max(M, N))."""
        a = {"cannon": 0, "tallskinny": 1, "auto": 2}.get(algorithm, algorithm)
        _check(load().dbm_ctx_set_algorithm(self.h, int(a)))
        self.algorithm = a

    def set_densify_threshold(self, threshold: float) -> None:
        """should_densify threshold of path='auto': densify iff occupancy >= threshold."""
        _check(load().dbm_ctx_set_densify_threshold(self.h, threshold))

    def set_dense_chunk_bytes(self, nbytes: int) -> None:
        _check(load().dbm_ctx_set_dense_chunk_bytes(self.h, nbytes))

    def launch_count(self) -> int:
        n = C.c_int64()
        _check(load().dbm_ctx_launch_count(self.h, C.byref(n)))
        return n.value

    def workspace(self, nbytes: int) -> torch.Tensor:
        """Caller-owned multiply workspace, cached and grown on demand (the paper's memory pool)."""
        if self._ws is None or self._ws.numel() < nbytes:
            self._ws = None
            self._ws = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=self.device)
        return self._ws

    def release_workspace(self) -> None:
        self._ws = None

    def close(self) -> None:
        if getattr(self, "h", None):
            load().dbm_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---------------------------------------------------------------------------- matrix
def pattern_random(seed: int, mat_id: int, Mb: int, Nb: int, occupancy: float):
    """dbm_pattern_random: (Mb, Nb) uint8 numpy mask of stored blocks (reading R15)."""
    import numpy as np

    m = np.empty(max(Mb * Nb, 1), dtype=np.uint8)
    _check(load().dbm_pattern_random(seed, mat_id, Mb, Nb, occupancy, m.ctypes.data))
    return m[: Mb * Nb].reshape(Mb, Nb)


def pattern_product(amask, bmask, cmask=None):
    """dbm_pattern_product: the product pattern of A's and B's masks OR-ed into cmask (fill-in workflow, R15)."""
    import numpy as np

    a = np.ascontiguousarray(amask, dtype=np.uint8)
    b = np.ascontiguousarray(bmask, dtype=np.uint8)
    Mb, Kb = a.shape
    Nb = b.shape[1]
    c = np.zeros((Mb, Nb), dtype=np.uint8) if cmask is None else np.array(cmask, dtype=np.uint8, order="C")
    _check(load().dbm_pattern_product(Mb, Kb, Nb, a.ctypes.data, b.ctypes.data, c.ctypes.data))
    return c


class Matrix:
    """dbm_matrix: rows x cols FP64 matrix of bs x bs blocks, block-cyclic over ctx's grid.
    mask (numpy (Mb, Nb), nonzero = stored) makes it block-sparse (dbm_matrix_create_sparse, R15)."""

    def __init__(self, ctx: Context, rows: int, cols: int, block_size: int, arena: torch.Tensor | None = None,
                 mask=None, sparse: bool = False, row_sizes=None, col_sizes=None):
        lib = load()
        h = C.c_void_p()
        self.sparse = sparse or mask is not None
        self.row_sizes = self.col_sizes = None
        if row_sizes is not None:  # non-uniform block sizes (dbm_matrix_create_blocked, reading R16)
            import numpy as np

            rs = np.ascontiguousarray(row_sizes, dtype=np.int32)
            cs = np.ascontiguousarray(col_sizes, dtype=np.int32)
            mk = None
            if mask is not None:
                mk = np.ascontiguousarray(mask, dtype=np.uint8)
                assert mk.size == rs.size * cs.size
            _check(lib.dbm_matrix_create_blocked(ctx.h, rs.size, rs.ctypes.data, cs.size, cs.ctypes.data,
                                                 mk.ctypes.data if mk is not None else None, C.byref(h)))
            rows, cols = int(rs.sum()), int(cs.sum())
            self.row_sizes, self.col_sizes = rs, cs
            block_size = int(rs[0]) if (rs.size and (rs == rs[0]).all() and (cs == rs[0]).all()) else 0
        elif self.sparse:
            import numpy as np

            mk = None
            if mask is not None:
                mk = np.ascontiguousarray(mask, dtype=np.uint8)
                assert mk.size == (rows // block_size) * (cols // block_size)
            _check(lib.dbm_matrix_create_sparse(ctx.h, rows, cols, block_size,
                                                mk.ctypes.data if mk is not None else None, C.byref(h)))
        else:
            _check(lib.dbm_matrix_create(ctx.h, rows, cols, block_size, C.byref(h)))
        self.h, self.ctx = h, ctx
        self.rows, self.cols, self.bs = rows, cols, block_size
        ml, nl, nb = C.c_int64(), C.c_int64(), C.c_int64()
        _check(lib.dbm_matrix_local_info(h, C.byref(ml), C.byref(nl), C.byref(nb)))
        self.mloc, self.nloc, self.arena_bytes = ml.value, nl.value, nb.value
        lo, gl = C.c_int64(), C.c_int64()
        _check(lib.dbm_matrix_nnz(h, C.byref(lo), C.byref(gl)))
        self.nnz, self.global_nnz = lo.value, gl.value
        if arena is None:
            arena = torch.empty(max(self.arena_bytes // 8, 2), dtype=torch.float64, device=ctx.device)
        self.arena = arena
        _check(lib.dbm_matrix_attach(h, arena.data_ptr(), arena.numel() * arena.element_size()))

    def fill_random(self, seed: int, mat_id: int, kind: int = 0) -> None:
        _check(load().dbm_matrix_fill_random(self.h, seed, mat_id, kind))

    def local_csr(self):
        import numpy as np

        rp = np.empty(self.mloc + 1, dtype=np.int64)
        ci = np.empty(max(self.nnz, 1), dtype=np.int64)
        ri = np.empty(max(self.mloc, 1), dtype=np.int64)
        _check(load().dbm_matrix_local_csr(self.h, rp.ctypes.data, ci.ctypes.data, ri.ctypes.data))
        return rp, ci[: self.nnz], ri[: self.mloc]

    def block_shape(self, bi: int, bj: int) -> tuple[int, int]:
        if self.row_sizes is None:
            return self.bs, self.bs
        return int(self.row_sizes[bi]), int(self.col_sizes[bj])

    def set_block(self, bi: int, bj: int, block) -> None:
        import numpy as np

        b = np.asfortranarray(np.asarray(block, dtype=np.float64))
        assert b.shape == self.block_shape(bi, bj)
        _check(load().dbm_matrix_set_block(self.h, bi, bj, b.ctypes.data))

    def get_block(self, bi: int, bj: int):
        import numpy as np

        b = np.empty(self.block_shape(bi, bj), dtype=np.float64, order="F")
        _check(load().dbm_matrix_get_block(self.h, bi, bj, b.ctypes.data))
        return b

    def upload(self, host: torch.Tensor) -> None:
        assert host.dtype == torch.float64 and host.numel() * 8 >= self.arena_bytes and host.is_contiguous()
        _check(load().dbm_matrix_upload(self.h, host.data_ptr()))

    def download(self, host: torch.Tensor) -> None:
        assert host.dtype == torch.float64 and host.numel() * 8 >= self.arena_bytes and host.is_contiguous()
        _check(load().dbm_matrix_download(self.h, host.data_ptr()))

    def owner_of_block(self, bi: int, bj: int) -> int:
        r = C.c_int()
        _check(load().dbm_owner_of_block(self.h, bi, bj, C.byref(r)))
        return r.value

    def local_view(self) -> torch.Tensor:
        """The arena as (mloc*nloc, bs, bs) blocks; block[.., x, y] -> use .transpose for column-major."""
        n = self.nnz * self.bs * self.bs
        return self.arena[:n]

    def local_dims(self) -> tuple[int, int]:
        """Element rows and columns of this rank's local share (sum of its block sizes)."""
        if self.row_sizes is None:
            return self.mloc * self.bs, self.nloc * self.bs
        c = self.ctx
        return int(self.row_sizes[c.myrow::c.pr].sum()), int(self.col_sizes[c.mycol::c.pc].sum())

    def densify(self, dense: torch.Tensor, ld: int | None = None, layout: int = 0) -> None:
        if ld is None:
            ld = self.local_dims()[0] if layout == 0 else self.local_dims()[1]
        _check(load().dbm_densify(self.h, dense.data_ptr(), ld, layout))

    def undensify(self, dense: torch.Tensor, alpha: float = 1.0, beta: float = 0.0, ld: int | None = None) -> None:
        if ld is None:
            ld = self.local_dims()[0]
        _check(load().dbm_undensify(self.h, dense.data_ptr(), ld, alpha, beta))

    def close(self) -> None:
        if getattr(self, "h", None):
            load().dbm_matrix_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---------------------------------------------------------------------------- multiply
def multiply_workspace(ctx: Context, A: Matrix, B: Matrix, C_: Matrix, path="densified") -> int:
    n = C.c_int64()
    _check(load().dbm_multiply_workspace(ctx.h, A.h, B.h, C_.h, _PATHS[path], C.byref(n)))
    return n.value


def multiply(ctx: Context, alpha: float, A: Matrix, B: Matrix, beta: float, C_: Matrix, path="densified",
             stack_cap: int = 0, workspace: torch.Tensor | None = None) -> dict:
    """C = alpha*A*B + beta*C (dbm_multiply): Cannon + blocked / densified local multiply."""
    lib = load()
    need = multiply_workspace(ctx, A, B, C_, path)
    ws = workspace if workspace is not None else ctx.workspace(need)
    st = Stats()
    _check(lib.dbm_multiply(ctx.h, alpha, A.h, B.h, beta, C_.h, _PATHS[path], stack_cap, ws.data_ptr(),
                            ws.numel() * ws.element_size(), C.byref(st)))
    return st.as_dict()


def debug_first_step(pr: int, pc: int, rank: int) -> int:
    """Host-only: the canonical Cannon step `rank` takes first under the copy-engine transport
    (dbm_debug_first_step, the local-first order)."""
    v = C.c_int(0)
    _check(load().dbm_debug_first_step(pr, pc, rank, C.byref(v)))
    return v.value


def plan_exchange(pr: int, pc: int, myrow: int, mycol: int, Mb: int, Nb: int, Kb: int, bs: int, step: int,
                  path="densified") -> list[dict]:
    """Host-only: the send/recv list dbm_multiply issues at Cannon step `step` (dbm_plan_exchange)."""
    import numpy as np

    lib = load()
    n = C.c_int(0)
    _check(lib.dbm_plan_exchange(pr, pc, myrow, mycol, Mb, Nb, Kb, bs, _PATHS[path], step, None, None, C.byref(n)))
    ops = np.zeros(4 * max(n.value, 1), dtype=np.int32)
    by = np.zeros(max(n.value, 1), dtype=np.int64)
    _check(lib.dbm_plan_exchange(pr, pc, myrow, mycol, Mb, Nb, Kb, bs, _PATHS[path], step, ops.ctypes.data,
                                 by.ctypes.data, C.byref(n)))
    return [{"send": bool(ops[4 * i]), "operand": "AB"[ops[4 * i + 1]], "peer": int(ops[4 * i + 2]),
             "kappa": int(ops[4 * i + 3]), "bytes": int(by[i])} for i in range(n.value)]


def multiply_host(ctx: Context, alpha: float, A: Matrix, B: Matrix, beta: float, C_: Matrix, A_host: torch.Tensor,
                  B_host: torch.Tensor, C_host: torch.Tensor, path="densified", stack_cap: int = 0,
                  workspace: torch.Tensor | None = None) -> dict:
    """dbm_multiply_host: C_host = alpha*A_host*B_host + beta*C_host with host-resident (ideally pinned)
    arenas streamed through the device matrices.  Asynchronous on the ctx stream."""
    for h, m in ((A_host, A), (B_host, B), (C_host, C_)):
        assert h.dtype == torch.float64 and h.is_contiguous() and h.numel() * 8 >= m.arena_bytes and not h.is_cuda
    lib = load()
    need = multiply_workspace(ctx, A, B, C_, path)
    ws = workspace if workspace is not None else ctx.workspace(need)
    st = Stats()
    _check(lib.dbm_multiply_host(ctx.h, alpha, A.h, B.h, beta, C_.h, _PATHS[path], stack_cap, ws.data_ptr(),
                                 ws.numel() * ws.element_size(), A_host.data_ptr(), B_host.data_ptr(),
                                 C_host.data_ptr(), C.byref(st)))
    return st.as_dict()


def plan_tallskinny(pr: int, pc: int, myrow: int, mycol: int, Mb: int, Nb: int, Kb: int, bs: int) -> tuple[int, int]:
    """Host-only: (bytes received, bytes sent) of rank (myrow, mycol) in one tall-and-skinny multiply."""
    rv, sd = C.c_int64(), C.c_int64()
    _check(load().dbm_plan_tallskinny(pr, pc, myrow, mycol, Mb, Nb, Kb, bs, C.byref(rv), C.byref(sd)))
    return rv.value, sd.value


def debug_stacks(ctx: Context, A: Matrix, B: Matrix, C_: Matrix, step: int = 0, cap: int = 0):
    import numpy as np

    lib = load()
    ne, ns = C.c_int64(), C.c_int64()
    _check(lib.dbm_debug_stacks(ctx.h, A.h, B.h, C_.h, step, cap, None, C.byref(ne), None, C.byref(ns)))
    trip = np.empty(max(3 * ne.value, 3), dtype=np.int32)
    ptr = np.empty(ns.value + 1, dtype=np.int64)
    _check(lib.dbm_debug_stacks(ctx.h, A.h, B.h, C_.h, step, cap, trip.ctypes.data, C.byref(ne), ptr.ctypes.data,
                                C.byref(ns)))
    return trip[: 3 * ne.value].reshape(ne.value, 3), ptr


def debug_pack_panel(m: Matrix, operand: int, first: int, stride: int, nk: int, out: torch.Tensor,
                     pitch: int = 0) -> None:
    """dbm_debug_pack_panel: pack nk local block columns (operand 0) / rows (operand 1) into `out`."""
    _check(load().dbm_debug_pack_panel(m.h, operand, first, stride, nk, pitch, out.data_ptr() if out.numel() else None))


def debug_dgemm(ctx: Context, M: int, N: int, K: int, alpha: float, At: torch.Tensor, lda: int, B: torch.Tensor,
                ldb: int, beta: float, Cm: torch.Tensor, ldc: int, splitk: int = 1,
                partial: torch.Tensor | None = None) -> None:
    pb = partial.numel() * partial.element_size() if partial is not None else 0
    _check(load().dbm_debug_dgemm(ctx.h, M, N, K, alpha, At.data_ptr(), lda, B.data_ptr(), ldb, beta,
                                  Cm.data_ptr(), ldc, splitk, partial.data_ptr() if partial is not None else None,
                                  pb))
