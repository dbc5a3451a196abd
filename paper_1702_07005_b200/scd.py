"""Thin Python binding of the C ABI in include/scd.h (argument marshalling only).

Every step of the hot path runs in libscd.so's CUDA kernels; this module only converts
arguments (torch CUDA tensors are passed as borrowed device pointers, numpy arrays as host
buffers that the library copies) and maps status codes to exceptions.  There is no CPU
fallback: if libscd.so is missing or CUDA is unavailable, calls raise.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

# SCD_LIBSCD: another build of the same library (A/B measurements of kernel changes, tools/)
_SO = os.environ.get("SCD_LIBSCD") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libscd.so")

PRIMAL, DUAL = 0, 1
AGG = {"add": 0, "average": 1, "optimal": 2}
MEM_HOST, MEM_DEVICE = 0, 1
CSR, CSC = 0, 1
STATUS = ["SCD_OK", "SCD_E_INVALID_ARG", "SCD_E_BAD_MATRIX", "SCD_E_OOM", "SCD_E_CUDA", "SCD_E_NCCL",
          "SCD_E_STATE", "SCD_E_UNSUPPORTED"]


class ScdError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS[status] if 0 <= status < len(STATUS) else status}: {msg}")
        self.status = status


class Matrix(C.Structure):
    _fields_ = [("layout", C.c_int), ("n_rows", C.c_int64), ("n_cols", C.c_int64), ("nnz", C.c_int64),
                ("ptr", C.c_void_p), ("idx", C.c_void_p), ("val", C.c_void_p), ("mem", C.c_int)]


# scd_collectives (include/scd.h): host-side transport hooks used instead of an NCCL communicator
DT_F32, DT_F64, DT_I32, DT_I64, DT_U8 = 0, 1, 2, 3, 4
OP_SUM, OP_MAX, OP_MIN = 0, 1, 2
ALLREDUCE_FN = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_int32, C.c_void_p)
ALLGATHER_FN = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p)


class Collectives(C.Structure):
    _fields_ = [("user", C.c_void_p), ("allreduce", ALLREDUCE_FN), ("allgather", ALLGATHER_FN)]


class Options(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("n_global", C.c_int64), ("rank", C.c_int32), ("world", C.c_int32),
                ("nccl_comm", C.c_void_p), ("stream", C.c_void_p), ("deterministic", C.c_int32),
                ("max_inflight", C.c_int32), ("recompute_every", C.c_int32), ("validate", C.c_int32),
                ("profile", C.c_int32), ("wild", C.c_int32), ("collectives", C.POINTER(Collectives)),
                ("block_order", C.c_int32)]


class Info(C.Structure):
    _fields_ = [("n_coord", C.c_int64), ("n_shared", C.c_int64), ("nnz", C.c_int64), ("n_nonempty", C.c_int64),
                ("n_bins", C.c_int32), ("bin_kind", C.c_int32 * 4), ("bin_count", C.c_int64 * 4),
                ("bin_nnz", C.c_int64 * 4), ("bin_grid", C.c_int32 * 4), ("bin_block", C.c_int32 * 4),
                ("launches", C.c_int64), ("tau_star", C.c_double), ("inflight_cap", C.c_int64),
                ("bin_cap", C.c_int64 * 4), ("bin_tau", C.c_double * 4), ("n_slices", C.c_int32),
                ("sv_offset_bytes", C.c_int64), ("probe_best_ms", C.c_float), ("probe_worst_ms", C.c_float),
                ("bin_head", C.c_int32 * 4), ("bin_flush", C.c_int32 * 4), ("bin_hot", C.c_int32 * 4),
                ("hot_cover", C.c_double), ("tail_snap", C.c_int32), ("tail_tau", C.c_double), ("bin_snap", C.c_int32 * 4), ("tail_roll", C.c_int64), ("head_copy", C.c_int64), ("hot_copy", C.c_int64), ("hot_tp", C.c_int32), ("hot_tail_tau", C.c_double), ("hot_hp", C.c_int32),
                ("sm_head", C.c_int32), ("sm_chunk", C.c_int32), ("sm_ch", C.c_int32), ("sm_rh", C.c_int32)]


_lib = None
EXPORTS = ("scd_default_options", "scd_create", "scd_epoch", "scd_epoch_part", "scd_objective", "scd_duality_gap", "scd_aggregate",
           "scd_aggregate_group", "scd_evaluate_group", "scd_get_model", "scd_get_shared", "scd_set_model", "scd_recompute_shared",
           "scd_get_stream", "scd_get_info", "scd_profile_read", "scd_last_error", "scd_last_global_error",
           "scd_status_string", "scd_struct_sizes", "scd_destroy", "scd_permutation", "scd_block_permutation", "scd_partition", "scd_partition_balanced", "scd_transpose", "scd_renumber", "scd_libsvm_size", "scd_libsvm_read",
           "scd_nccl_unique_id", "scd_nccl_comm_init", "scd_nccl_comm_destroy")


def lib():
    """Load libscd.so (raises if it was not built: there is no fallback path)."""
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            raise ImportError(f"{_SO} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(_SO)
        V, P, I64, I32, U32, D = C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_uint32, C.c_double
        sig = {
            "scd_default_options": (None, [C.POINTER(Options)]),
            "scd_create": (C.c_int, [C.POINTER(Matrix), P, C.c_int, D, C.c_int, C.POINTER(Options), C.POINTER(V)]),
            "scd_epoch": (C.c_int, [V, U32]),
            "scd_epoch_part": (C.c_int, [V, U32, I32, I32]),
            "scd_objective": (C.c_int, [V, C.POINTER(D), C.POINTER(D)]),
            "scd_duality_gap": (C.c_int, [V, C.POINTER(D)]),
            "scd_aggregate": (C.c_int, [V, C.c_int, C.POINTER(D)]),
            "scd_aggregate_group": (C.c_int, [P, I32, C.c_int, C.POINTER(D)]),
            "scd_evaluate_group": (C.c_int, [P, I32, C.POINTER(D), C.POINTER(D), C.POINTER(D)]),
            "scd_get_model": (C.c_int, [V, P, I64]),
            "scd_get_shared": (C.c_int, [V, P, I64]),
            "scd_set_model": (C.c_int, [V, P, I64]),
            "scd_recompute_shared": (C.c_int, [V]),
            "scd_get_stream": (C.c_int, [V, C.POINTER(V)]),
            "scd_get_info": (C.c_int, [V, C.POINTER(Info)]),
            "scd_profile_read": (C.c_int, [V, P, P, I32, C.POINTER(I32)]),
            "scd_last_error": (C.c_char_p, [V]),
            "scd_last_global_error": (C.c_char_p, []),
            "scd_status_string": (C.c_char_p, [C.c_int]),
            "scd_struct_sizes": (None, [P]),
            "scd_destroy": (None, [V]),
            "scd_permutation": (C.c_int, [C.c_uint64, U32, U32, I64, P]),
            "scd_block_permutation": (C.c_int, [C.c_uint64, U32, U32, I64, I64, P]),
            "scd_partition": (C.c_int, [C.c_uint64, I64, I32, P]),
            "scd_partition_balanced": (C.c_int, [P, I64, C.c_int, C.c_uint64, I32, P]),
            "scd_transpose": (C.c_int, [C.POINTER(Matrix), P, P, P, C.c_int]),
            "scd_renumber": (C.c_int, [C.POINTER(Matrix), P, P, P, P, C.c_int]),
            "scd_libsvm_size": (C.c_int, [C.c_char_p, I64, C.POINTER(I64), C.POINTER(I64), C.POINTER(I64)]),
            "scd_libsvm_read": (C.c_int, [C.c_char_p, I64, P, P, P, P]),
            "scd_nccl_unique_id": (C.c_int, [P]),
            "scd_nccl_comm_init": (C.c_int, [P, I32, I32, C.POINTER(V)]),
            "scd_nccl_comm_destroy": (C.c_int, [V]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _check(st: int, ctx=None):
    if st != 0:
        L = lib()
        msg = (L.scd_last_error(ctx) if ctx else L.scd_last_global_error()) or b""
        raise ScdError(st, msg.decode(errors="replace"))


def _is_torch(a) -> bool:
    return type(a).__module__.startswith("torch")


def _buf(a, dtype):
    """-> (pointer, mem, keepalive).  torch CUDA tensors are borrowed device memory; everything
    else becomes a contiguous numpy array of ``dtype`` in host memory."""
    if _is_torch(a):
        import torch

        tdt = {np.int64: torch.int64, np.int32: torch.int32, np.float32: torch.float32}[dtype]
        if a.dtype != tdt or not a.is_contiguous():
            raise TypeError(f"tensor must be contiguous {tdt}, got {a.dtype}")
        if a.is_cuda:
            return a.data_ptr(), MEM_DEVICE, a
        a = a.numpy()
    arr = np.ascontiguousarray(a, dtype=dtype)
    return arr.ctypes.data, MEM_HOST, arr


class Solver:
    """One TPA-SCD context (scd_create ... scd_destroy).

    form='dual' takes A in CSR (by example), form='primal' A in CSC (by feature): ``ptr``,
    ``idx``, ``val`` are the outer offsets / inner indices / values of that layout."""

    def __init__(self, ptr, idx, val, n_rows: int, n_cols: int, y, lam: float, form: str = "dual", *,
                 seed: int = 0, deterministic: bool = False, max_inflight: int = 0, n_global: int = 0,
                 rank: int = 0, world: int = 1, nccl_comm=None, stream=None, validate: bool = True,
                 profile: bool = False, recompute_every: int = 0, wild: bool = False,
                 collectives: Collectives | None = None, block_order: int = 0):
        L = lib()
        self._form = PRIMAL if form == "primal" else DUAL
        if form not in ("primal", "dual"):
            raise ValueError(form)
        p, mp, kp = _buf(ptr, np.int64)
        i, mi, ki = _buf(idx, np.int32)
        # val=None: implicit values 1.0f (one-hot data, P:460 footnote)
        v, mv, kv = _buf(val, np.float32) if val is not None else (None, mp, None)
        if not (mp == mi == mv):
            raise ValueError("ptr/idx/val must all be host arrays or all CUDA tensors")
        yy, my, ky = _buf(y, np.float32)
        nnz = int(kp[-1]) if mp == MEM_HOST else int(kp[-1].item())
        self._keep = (kp, ki, kv, ky, collectives)
        m = Matrix(CSC if self._form == PRIMAL else CSR, n_rows, n_cols, nnz, p, i, v, mp)
        o = Options()
        L.scd_default_options(C.byref(o))
        o.seed = seed & (2**64 - 1)
        o.n_global = n_global
        o.rank, o.world = rank, world
        o.nccl_comm = nccl_comm
        o.stream = None if stream is None else (stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))
        o.deterministic = int(deterministic)
        o.max_inflight = max_inflight
        o.recompute_every = recompute_every
        o.validate = int(validate)
        o.profile = int(profile)
        o.wild = int(wild)
        o.block_order = int(block_order)
        if collectives is not None:  # borrowed by the context: kept alive with it
            o.collectives = C.pointer(collectives)
        h = C.c_void_p()
        _check(L.scd_create(C.byref(m), yy, my, float(lam), self._form, C.byref(o), C.byref(h)))
        self._h = h
        self.n_rows, self.n_cols, self.nnz, self.lam = n_rows, n_cols, nnz, lam
        self.n_coord = n_cols if self._form == PRIMAL else n_rows
        self.n_shared = n_rows if self._form == PRIMAL else n_cols

    # --- hot path -----------------------------------------------------------------------------
    def epoch(self, t: int):
        _check(lib().scd_epoch(self._h, t & 0xFFFFFFFF), self._h)

    def epoch_part(self, t: int, part: int, nparts: int):
        """Part `part` of `nparts` of epoch t (sub-epoch aggregation rounds)."""
        _check(lib().scd_epoch_part(self._h, t & 0xFFFFFFFF, part, nparts), self._h)

    def objective(self) -> tuple[float, float]:
        P, D = C.c_double(), C.c_double()
        _check(lib().scd_objective(self._h, C.byref(P), C.byref(D)), self._h)
        return P.value, D.value

    def duality_gap(self) -> float:
        g = C.c_double()
        _check(lib().scd_duality_gap(self._h, C.byref(g)), self._h)
        return g.value

    def aggregate(self, mode: str = "optimal") -> float:
        g = C.c_double()
        _check(lib().scd_aggregate(self._h, AGG[mode], C.byref(g)), self._h)
        return g.value

    # --- state ---------------------------------------------------------------------------------
    def get_model(self) -> np.ndarray:
        out = np.empty(self.n_coord, np.float32)
        _check(lib().scd_get_model(self._h, out.ctypes.data, self.n_coord), self._h)
        return out

    def get_shared(self) -> np.ndarray:
        out = np.empty(self.n_shared, np.float32)
        _check(lib().scd_get_shared(self._h, out.ctypes.data, self.n_shared), self._h)
        return out

    def set_model(self, x):
        x = np.ascontiguousarray(x, np.float32)
        _check(lib().scd_set_model(self._h, x.ctypes.data, len(x)), self._h)

    def recompute_shared(self):
        _check(lib().scd_recompute_shared(self._h), self._h)

    @property
    def stream_handle(self) -> int:
        s = C.c_void_p()
        _check(lib().scd_get_stream(self._h, C.byref(s)), self._h)
        return s.value or 0

    def info(self) -> dict:
        inf = Info()
        _check(lib().scd_get_info(self._h, C.byref(inf)), self._h)
        nb = inf.n_bins
        return dict(n_coord=inf.n_coord, n_shared=inf.n_shared, nnz=inf.nnz, n_nonempty=inf.n_nonempty,
                    launches=inf.launches, tau_star=inf.tau_star, inflight_cap=inf.inflight_cap,
                    n_slices=inf.n_slices, sv_offset_bytes=inf.sv_offset_bytes,
                    probe_ms=(inf.probe_best_ms, inf.probe_worst_ms), hot_cover=inf.hot_cover, tail_snap=inf.tail_snap,
                    tail_tau=inf.tail_tau, tail_roll=inf.tail_roll, head_copy=inf.head_copy, hot_copy=inf.hot_copy, hot_tp=inf.hot_tp, hot_tail_tau=inf.hot_tail_tau, hot_hp=inf.hot_hp,
                    sm_head=inf.sm_head, sm_chunk=inf.sm_chunk, sm_ch=inf.sm_ch, sm_rh=inf.sm_rh,
                    bins=[dict(lanes=inf.bin_kind[i], count=inf.bin_count[i], nnz=inf.bin_nnz[i],
                               grid=inf.bin_grid[i], block=inf.bin_block[i], cap=inf.bin_cap[i],
                               tau=inf.bin_tau[i], head=inf.bin_head[i], flush=inf.bin_flush[i],
                               hot=inf.bin_hot[i], snap=inf.bin_snap[i])
                          for i in range(nb)])

    def profile_read(self) -> list[tuple[float, int]]:
        ms = (C.c_double * 4)()
        cnt = (C.c_int64 * 4)()
        n = C.c_int32()
        _check(lib().scd_profile_read(self._h, ms, cnt, 4, C.byref(n)), self._h)
        return [(ms[i], cnt[i]) for i in range(n.value)]

    def close(self):
        if getattr(self, "_h", None):
            lib().scd_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


def aggregate_group(solvers, mode: str = "optimal") -> float:
    arr = (C.c_void_p * len(solvers))(*[s._h.value for s in solvers])
    g = C.c_double()
    _check(lib().scd_aggregate_group(arr, len(solvers), AGG[mode], C.byref(g)))
    return g.value


def evaluate_group(solvers) -> tuple[float, float, float]:
    """(P, D, gap) of the global model of logical workers on one device."""
    arr = (C.c_void_p * len(solvers))(*[s._h.value for s in solvers])
    P, D, g = C.c_double(), C.c_double(), C.c_double()
    _check(lib().scd_evaluate_group(arr, len(solvers), C.byref(P), C.byref(D), C.byref(g)))
    return P.value, D.value, g.value


def permutation(seed: int, epoch: int, n: int, stream: int = 0) -> np.ndarray:
    out = np.empty(max(n, 1), np.int64)
    _check(lib().scd_permutation(seed & (2**64 - 1), epoch, stream, n, out.ctypes.data))
    return out[:n]


def block_permutation(seed: int, epoch: int, n: int, blk: int, stream: int = 0) -> np.ndarray:
    out = np.empty(max(n, 1), np.int64)
    _check(lib().scd_block_permutation(seed & (2**64 - 1), epoch, stream, n, blk, out.ctypes.data))
    return out[:n]


def partition(seed: int, count: int, k: int) -> np.ndarray:
    out = np.empty(max(count, 1), np.int32)
    _check(lib().scd_partition(seed & (2**64 - 1), count, k, out.ctypes.data))
    return out[:count]


def partition_balanced(ptr, seed: int, k: int) -> np.ndarray:
    """Stored-entry balanced partition of the outer coordinates of ptr (scd_partition_balanced)."""
    p, mp, kp = _buf(ptr, np.int64)
    n = (len(kp) if mp == MEM_HOST else kp.numel()) - 1
    out = np.empty(max(n, 1), np.int32)
    _check(lib().scd_partition_balanced(p, n, mp, seed & (2**64 - 1), k, out.ctypes.data))
    return out[:n]


def transpose(ptr, idx, val, n_rows: int, n_cols: int, layout: str = "csr"):
    """Stable CSR<->CSC transpose on the device.  Host inputs -> numpy outputs; CUDA tensors ->
    CUDA tensors.  Returns (ptr, idx, val) of the other layout."""
    p, mp, kp = _buf(ptr, np.int64)
    i, mi, ki = _buf(idx, np.int32)
    v, mv, kv = _buf(val, np.float32) if val is not None else (None, mp, None)
    lay = CSR if layout == "csr" else CSC
    inner = n_cols if lay == CSR else n_rows
    nnz = int(kp[-1]) if mp == MEM_HOST else int(kp[-1].item())
    m = Matrix(lay, n_rows, n_cols, nnz, p, i, v, mp)
    if mp == MEM_DEVICE:
        import torch

        dev = kp.device
        op = torch.empty(inner + 1, dtype=torch.int64, device=dev)
        oi = torch.empty(max(nnz, 1), dtype=torch.int32, device=dev)
        ov = torch.empty(max(nnz, 1), dtype=torch.float32, device=dev)
        _check(lib().scd_transpose(C.byref(m), op.data_ptr(), oi.data_ptr(), ov.data_ptr(), MEM_DEVICE))
        return op, oi[:nnz], (ov[:nnz] if v is not None else None)
    op = np.empty(inner + 1, np.int64)
    oi = np.empty(max(nnz, 1), np.int32)
    ov = np.empty(max(nnz, 1), np.float32)
    _check(lib().scd_transpose(C.byref(m), op.ctypes.data, oi.ctypes.data, ov.ctypes.data, MEM_HOST))
    return op, oi[:nnz], (ov[:nnz] if v is not None else None)


def renumber(ptr, idx, val, n_rows: int, n_cols: int, layout: str = "csr"):
    """Renumber the inner indices by frequency on the device (scd_renumber).  Host inputs -> numpy
    outputs, CUDA tensors -> CUDA tensors.  Returns (ptr, idx, val, new_of_old)."""
    p, mp, kp = _buf(ptr, np.int64)
    i, mi, ki = _buf(idx, np.int32)
    v, mv, kv = _buf(val, np.float32) if val is not None else (None, mp, None)
    lay = CSR if layout == "csr" else CSC
    outer, inner = (n_rows, n_cols) if lay == CSR else (n_cols, n_rows)
    nnz = int(kp[-1]) if mp == MEM_HOST else int(kp[-1].item())
    m = Matrix(lay, n_rows, n_cols, nnz, p, i, v, mp)
    if mp == MEM_DEVICE:
        import torch

        dev = kp.device
        op = torch.empty(outer + 1, dtype=torch.int64, device=dev)
        oi = torch.empty(max(nnz, 1), dtype=torch.int32, device=dev)
        ov = torch.empty(max(nnz, 1), dtype=torch.float32, device=dev)
        om = torch.empty(inner, dtype=torch.int32, device=dev)
        _check(lib().scd_renumber(C.byref(m), op.data_ptr(), oi.data_ptr(), ov.data_ptr(), om.data_ptr(), MEM_DEVICE))
        return op, oi[:nnz], (ov[:nnz] if v is not None else None), om
    op = np.empty(outer + 1, np.int64)
    oi = np.empty(max(nnz, 1), np.int32)
    ov = np.empty(max(nnz, 1), np.float32)
    om = np.empty(inner, np.int32)
    _check(lib().scd_renumber(C.byref(m), op.ctypes.data, oi.ctypes.data, ov.ctypes.data, om.ctypes.data, MEM_HOST))
    return op, oi[:nnz], (ov[:nnz] if v is not None else None), om


def load_libsvm(path: str, n_cols: int | None = None) -> dict:
    """Read a LIBSVM text file into host CSR arrays (scd_libsvm_size + scd_libsvm_read):
    dict(ptr, idx, val, y, n_rows, n_cols) with 0-based indices."""
    L = lib()
    hint = int(n_cols or 0)
    r, z, c = C.c_int64(), C.c_int64(), C.c_int64()
    _check(L.scd_libsvm_size(path.encode(), hint, C.byref(r), C.byref(z), C.byref(c)))
    ptr = np.empty(r.value + 1, np.int64)
    idx = np.empty(max(z.value, 1), np.int32)
    val = np.empty(max(z.value, 1), np.float32)
    y = np.empty(max(r.value, 1), np.float32)
    _check(L.scd_libsvm_read(path.encode(), hint, ptr.ctypes.data, idx.ctypes.data, val.ctypes.data, y.ctypes.data))
    return dict(ptr=ptr, idx=idx[:z.value], val=val[:z.value], y=y[:r.value], n_rows=r.value, n_cols=c.value)


def nccl_unique_id() -> bytes:
    buf = (C.c_char * 128)()
    _check(lib().scd_nccl_unique_id(buf))
    return bytes(buf)


def nccl_comm_init(uid: bytes, world: int, rank: int) -> int:
    buf = (C.c_char * 128).from_buffer_copy(uid)
    h = C.c_void_p()
    _check(lib().scd_nccl_comm_init(buf, world, rank, C.byref(h)))
    return h.value


def nccl_comm_destroy(h: int):
    _check(lib().scd_nccl_comm_destroy(h))
