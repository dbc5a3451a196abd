"""ctypes loader for oracle/liboracle.so (TEST INFRASTRUCTURE ONLY; see oracle/__init__.py)."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_SO = os.path.join(os.path.dirname(os.path.abspath(__file__)), "liboracle.so")
_lib = None

_P = C.c_void_p
_I64 = C.c_int64
_D = C.c_double


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            raise RuntimeError(f"{_SO} missing: run __graft_entry__.build()")
        L = C.CDLL(_SO)
        L.orc_perm_key.restype = C.c_uint64
        L.orc_perm_key.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32]
        L.orc_perm_at.restype = C.c_int64
        L.orc_perm_at.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, _I64, _I64]
        L.orc_permutation.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, _I64, _P]
        L.orc_partition.argtypes = [C.c_uint64, _I64, C.c_int32, _P]
        L.orc_block_order.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, _I64, _I64, _P]
        L.orc_transpose.argtypes = [_I64, _I64, _P, _P, _P, _P, _P, _P]
        L.orc_sq_norms.argtypes = [_I64, _P, _P, _P]
        L.orc_primal_epoch.argtypes = [_I64, _P, _P, _P, _P, _D, _D, _P, _P, _P, _P, _I64, _P]
        L.orc_dual_epoch.argtypes = [_P, _P, _P, _P, _D, _I64, _P, _P, _P, _P, _I64, _P]
        _lib = L
    return _lib


def p(a: np.ndarray | None):
    return None if a is None else a.ctypes.data


def c64(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def perm_at(seed: int, epoch: int, stream: int, n: int, j: int) -> int:
    return int(lib().orc_perm_at(seed & (2**64 - 1), epoch, stream, n, j))


def permutation(seed: int, epoch: int, n: int, stream: int = 0) -> np.ndarray:
    """P_epoch over [0, n) (DESIGN.md c8), int64."""
    out = np.empty(max(n, 1), np.int64)
    lib().orc_permutation(seed & (2**64 - 1), epoch, stream, n, p(out))
    return out[:n]


def block_order(seed: int, epoch: int, n: int, blk: int, stream: int = 0) -> np.ndarray:
    """Epoch visiting order in blocks of blk consecutive coordinates (DESIGN.md c28), int64."""
    if blk < 1:
        raise ValueError("blk must be >= 1")
    out = np.empty(max(n, 1), np.int64)
    lib().orc_block_order(seed & (2**64 - 1), epoch, stream, n, blk, p(out))
    return out[:n]


def partition(seed: int, count: int, k: int) -> np.ndarray:
    """owner[c] for c in [0, count) (DESIGN.md c15), int32."""
    if k < 1:
        raise ValueError("k must be >= 1")
    out = np.empty(max(count, 1), np.int32)
    lib().orc_partition(seed & (2**64 - 1), count, k, p(out))
    return out[:count]


def partition_balanced(ptr, seed: int, k: int) -> np.ndarray:
    """Stored-entry balanced partition (reading c29): the outer
    coordinates sorted by decreasing length, ties by their position in the partition permutation
    (stream 0x50415254, epoch 0, as in partition()), dealt in snake order 0..k-1, k-1..0, ...;
    owner[c] for c in [0, n), int32."""
    if k < 1:
        raise ValueError("k must be >= 1")
    ptr = np.asarray(ptr, np.int64)
    n = len(ptr) - 1
    lens = np.diff(ptr)
    pos = np.empty(n, np.int64)
    pos[permutation(seed, 0, n, stream=0x50415254)] = np.arange(n)
    order = np.lexsort((pos, -lens))  # primary key: length descending; then position
    i = np.arange(n)
    r, j = i // k, i % k
    owner = np.empty(n, np.int32)
    owner[order] = np.where(r % 2 == 1, k - 1 - j, j)
    return owner


def transpose(ptr, idx, val, n_inner: int):
    """Stable CSR<->CSC transpose; returns (optr int64, oidx int32, oval float32)."""
    ptr, idx, val = c64(ptr, np.int64), c64(idx, np.int32), c64(val, np.float32)
    n_outer = len(ptr) - 1
    nnz = int(ptr[-1])
    optr = np.empty(n_inner + 1, np.int64)
    oidx = np.empty(max(nnz, 1), np.int32)
    oval = np.empty(max(nnz, 1), np.float32)
    lib().orc_transpose(n_outer, n_inner, p(ptr), p(idx), p(val), p(optr), p(oidx), p(oval))
    return optr, oidx[:nnz], oval[:nnz]


def sq_norms(ptr, val) -> np.ndarray:
    ptr, val = c64(ptr, np.int64), c64(val, np.float32)
    out = np.empty(max(len(ptr) - 1, 1), np.float64)
    lib().orc_sq_norms(len(ptr) - 1, p(ptr), p(val), p(out))
    return out[: len(ptr) - 1]
