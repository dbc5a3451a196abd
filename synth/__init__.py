"""Seeded synthetic input generators shared by the oracle side and the CUDA side.

Test/bench infrastructure only.  Holds none of the method's arithmetic: it produces
A (CSR: int64 ptr, int32 idx, float32 val) and labels y from a seed, with the shapes of
the paper's workloads (§III.D l.254 webspam; §V.B l.460 criteo).  The recipe for
each config is in DESIGN.md §3.  Host twin: ``libsynth_host.so`` (C, OpenMP);
device twin: ``libsynth_cuda.so`` (CUDA); the two are bit-exact (tests/test_synth*.py).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from functools import lru_cache

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_HOST_SO = os.path.join(_HERE, "libsynth_host.so")
_CUDA_SO = os.path.join(_HERE, "libsynth_cuda.so")

LEN_TABLE = 1024


class _ZipfRows(C.Structure):
    _fields_ = [("n_rows", C.c_int64), ("n_cols", C.c_int64), ("n_active", C.c_int64),
                ("seed", C.c_uint64), ("values_one", C.c_int32), ("flip_mask", C.c_int32),
                ("len_table", C.c_void_p), ("alias_thr", C.c_void_p), ("alias_idx", C.c_void_p)]


class _Fields(C.Structure):
    _fields_ = [("n_rows", C.c_int64), ("n_cols", C.c_int64), ("n_fields", C.c_int32),
                ("flip_mask", C.c_int32), ("seed", C.c_uint64), ("field_off", C.c_void_p),
                ("field_card", C.c_void_p), ("alias_thr", C.c_void_p), ("alias_idx", C.c_void_p)]


_host = None
_cuda = None


def _lib_host():
    global _host
    if _host is None:
        if not os.path.exists(_HOST_SO):
            raise RuntimeError(f"{_HOST_SO} missing: run __graft_entry__.build()")
        lib = C.CDLL(_HOST_SO)
        lib.synth_build_alias.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]
        lib.synth_zipf_row_lengths.argtypes = [C.POINTER(_ZipfRows), C.c_int64, C.c_int64, C.c_void_p]
        lib.synth_zipf_fill.argtypes = [C.POINTER(_ZipfRows), C.c_int64, C.c_int64, C.c_void_p,
                                        C.c_void_p, C.c_void_p, C.c_void_p, C.c_int]
        lib.synth_fields_fill.argtypes = [C.POINTER(_Fields), C.c_int64, C.c_int64, C.c_void_p,
                                          C.c_void_p, C.c_void_p, C.c_int]
        _host = lib
    return _host


def _lib_cuda():
    global _cuda
    if _cuda is None:
        if not os.path.exists(_CUDA_SO):
            raise RuntimeError(f"{_CUDA_SO} missing: run __graft_entry__.build()")
        lib = C.CDLL(_CUDA_SO)
        lib.synth_zipf_fill_device.argtypes = [C.POINTER(_ZipfRows), C.c_int64, C.c_int64, C.c_void_p,
                                               C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        lib.synth_fields_fill_device.argtypes = [C.POINTER(_Fields), C.c_int64, C.c_int64, C.c_void_p,
                                                 C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        _cuda = lib
    return _cuda


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


# ----------------------------------------------------------------------------- tables
@lru_cache(maxsize=16)
def zipf_alias(n: int, s: float) -> tuple[np.ndarray, np.ndarray]:
    """Alias table for P(f) ∝ (f+1)^-s over [0, n) (host, fp64 Vose; shared by both twins)."""
    w = np.power(np.arange(1, n + 1, dtype=np.float64), -float(s))
    thr = np.empty(n, np.uint32)
    ali = np.empty(n, np.uint32)
    rc = _lib_host().synth_build_alias(_ptr(w), n, _ptr(thr), _ptr(ali))
    if rc:
        raise RuntimeError(f"synth_build_alias failed rc={rc}")
    return thr, ali


@lru_cache(maxsize=16)
def lognormal_len_table(mean: float, sigma: float, lo: int, hi: int) -> np.ndarray:
    """1024-quantile table of a lognormal(mu, sigma) clamped to [lo, hi], mu solved so the
    table mean equals ``mean`` (rounded to integers).  sigma = 0 gives a constant table."""
    from scipy.special import ndtri

    z = ndtri((np.arange(LEN_TABLE) + 0.5) / LEN_TABLE)

    def table(mu):
        return np.clip(np.rint(np.exp(mu + sigma * z)), lo, hi)

    a, b = np.log(lo) - 5 * sigma - 1, np.log(hi) + 5 * sigma + 1
    for _ in range(200):
        m = 0.5 * (a + b)
        if table(m).mean() < mean:
            a = m
        else:
            b = m
    return table(0.5 * (a + b)).astype(np.uint32)


# ----------------------------------------------------------------------------- configs
@dataclass(frozen=True)
class ZipfRowsCfg:
    """Row-wise Zipf ("webspam-shaped") synthetic matrix; DESIGN.md §3."""
    name: str
    n_rows: int
    n_cols: int
    n_active: int
    zipf_s: float
    len_mean: float
    len_sigma: float
    len_lo: int
    len_hi: int
    seed: int
    values_one: bool = False
    flip_mask: int = 15
    lam: float = 1e-3

    def tables(self):
        thr, ali = zipf_alias(self.n_active, self.zipf_s)
        lt = lognormal_len_table(self.len_mean, self.len_sigma, self.len_lo, self.len_hi)
        return lt, thr, ali

    def struct(self):
        lt, thr, ali = self.tables()
        st = _ZipfRows(self.n_rows, self.n_cols, self.n_active, self.seed & (2**64 - 1),
                       int(self.values_one), self.flip_mask, _ptr(lt), _ptr(thr), _ptr(ali))
        return st, (lt, thr, ali)

    def with_rows(self, n_rows: int, name: str | None = None) -> "ZipfRowsCfg":
        d = dict(self.__dict__)
        d["n_rows"] = n_rows
        d["name"] = name or f"{self.name}[:{n_rows}]"
        return ZipfRowsCfg(**d)


@dataclass(frozen=True)
class FieldsCfg:
    """One-hot field ("criteo-shaped") synthetic matrix; DESIGN.md §3."""
    name: str
    n_rows: int
    cards: tuple
    zipf_s: float
    seed: int
    flip_mask: int = 15
    lam: float = 1e-3

    @property
    def n_cols(self) -> int:
        return int(sum(self.cards))

    @property
    def offsets(self) -> np.ndarray:
        return np.concatenate([[0], np.cumsum(np.asarray(self.cards, np.int64))[:-1]]).astype(np.int64)

    def tables(self):
        return _fields_alias(self.cards, self.zipf_s)

    def struct(self):
        thr, ali = self.tables()
        off = self.offsets
        card = np.asarray(self.cards, np.int64)
        st = _Fields(self.n_rows, self.n_cols, len(self.cards), self.flip_mask, self.seed & (2**64 - 1),
                     _ptr(off), _ptr(card), _ptr(thr), _ptr(ali))
        return st, (off, card, thr, ali)

    def with_rows(self, n_rows: int, name: str | None = None) -> "FieldsCfg":
        d = dict(self.__dict__)
        d["n_rows"] = n_rows
        d["name"] = name or f"{self.name}[:{n_rows}]"
        return FieldsCfg(**d)


@lru_cache(maxsize=4)
def _fields_alias(cards: tuple, s: float):
    thr = np.empty(int(sum(cards)), np.uint32)
    ali = np.empty(int(sum(cards)), np.uint32)
    off = 0
    for c in cards:
        t, a = zipf_alias(int(c), s) if c > 1 else (np.full(1, 0xFFFFFFFF, np.uint32), np.zeros(1, np.uint32))
        thr[off:off + c] = t
        ali[off:off + c] = a
        off += c
    zipf_alias.cache_clear()
    return thr, ali


@dataclass(frozen=True)
class DenseCfg:
    """Dense Gaussian ridge problem (config C1): A ~ N(0,1), y = A beta~ + 0.1 eps (numpy PCG64)."""
    name: str
    n_rows: int
    n_cols: int
    seed: int
    lam: float = 1e-3


_CRITEO_CAT = (20_000_000, 15_000_000, 10_000_000, 8_000_000, 6_000_000, 5_000_000, 4_000_000,
               3_000_000, 2_000_000, 1_000_000, 500_000, 300_000, 200_000, 100_000, 50_000, 20_000,
               10_000, 5_000, 2_000, 1_000, 500, 200, 100, 50, 20, 10)


def criteo_cards(total: int = 75_000_000, scale: float = 1.0) -> tuple:
    """13 numeric fields x 64 buckets + 26 categorical fields, rescaled so the sum is ``total``."""
    cat = np.asarray(_CRITEO_CAT, np.float64)
    num = 13 * 64
    cat = cat * ((total - num) / cat.sum()) * scale
    cat = np.maximum(1, np.floor(cat)).astype(np.int64)
    if scale == 1.0:
        cat[0] += total - num - int(cat.sum())
    return tuple([64] * 13 + [int(c) for c in cat])


CONFIGS = {
    # BASELINE.json configs[0..4]; seeds 1..5.
    "C1": DenseCfg("C1", 1000, 100, seed=1, lam=1e-3),
    "C2": ZipfRowsCfg("C2", 100_000, 50_000, 50_000, 1.0, 500.0, 0.5, 16, 5000, seed=2),
    "C3": ZipfRowsCfg("C3", 350_000, 16_609_143, 680_715, 1.0, 3728.0, 0.6, 64, 16384, seed=3),
    "C5": FieldsCfg("C5", 200_000_000, criteo_cards(), 1.1, seed=5),
}
# C4 is C3's matrix in CSC, partitioned by feature.


def c5_scaled(n_rows: int, scale: float) -> FieldsCfg:
    """Criteo-shaped problem with field cardinalities scaled by ``scale`` (tests)."""
    return FieldsCfg(f"C5x{scale:g}", n_rows, criteo_cards(75_000_000, scale), 1.1, seed=5)


# ----------------------------------------------------------------------------- host twin
def row_lengths(cfg, row0: int = 0, nrows: int | None = None) -> np.ndarray:
    nrows = cfg.n_rows - row0 if nrows is None else nrows
    if isinstance(cfg, FieldsCfg):
        return np.full(nrows, len(cfg.cards), np.int64)
    st, keep = cfg.struct()
    out = np.empty(nrows, np.int64)
    _lib_host().synth_zipf_row_lengths(C.byref(st), row0, nrows, _ptr(out))
    return out


def gen_host(cfg, row0: int = 0, nrows: int | None = None, threads: int = 0) -> dict:
    """Generate rows [row0, row0+nrows) on the host: dict(ptr, idx, val, y, n_rows, n_cols, lam)."""
    if isinstance(cfg, DenseCfg):
        return dense_gaussian(cfg)
    nrows = cfg.n_rows - row0 if nrows is None else nrows
    lens = row_lengths(cfg, row0, nrows)
    ptr = np.zeros(nrows + 1, np.int64)
    np.cumsum(lens, out=ptr[1:])
    nnz = int(ptr[-1])
    idx = np.empty(max(nnz, 1), np.int32)
    val = np.empty(max(nnz, 1), np.float32)
    y = np.empty(max(nrows, 1), np.float32)
    st, keep = cfg.struct()
    if isinstance(cfg, FieldsCfg):
        rc = _lib_host().synth_fields_fill(C.byref(st), row0, nrows, _ptr(idx), _ptr(val), _ptr(y), threads)
    else:
        rc = _lib_host().synth_zipf_fill(C.byref(st), row0, nrows, _ptr(ptr), _ptr(idx), _ptr(val), _ptr(y),
                                         threads)
    if rc:
        raise RuntimeError(f"synth host fill failed rc={rc}")
    return dict(ptr=ptr, idx=idx[:nnz], val=val[:nnz], y=y[:nrows], n_rows=nrows, n_cols=cfg.n_cols,
                lam=cfg.lam, name=cfg.name)


def dense_gaussian(cfg: DenseCfg) -> dict:
    rng = np.random.Generator(np.random.PCG64(cfg.seed))
    A = rng.standard_normal((cfg.n_rows, cfg.n_cols)).astype(np.float32)
    bt = rng.standard_normal(cfg.n_cols)
    y = (A.astype(np.float64) @ bt + 0.1 * rng.standard_normal(cfg.n_rows)).astype(np.float32)
    ptr = (np.arange(cfg.n_rows + 1, dtype=np.int64) * cfg.n_cols)
    idx = np.tile(np.arange(cfg.n_cols, dtype=np.int32), cfg.n_rows)
    return dict(ptr=ptr, idx=idx, val=A.ravel().copy(), y=y, n_rows=cfg.n_rows, n_cols=cfg.n_cols,
                lam=cfg.lam, name=cfg.name)


def random_sparse(n_rows: int, n_cols: int, density: float, seed: int, empty_rows: int = 0,
                  empty_cols: int = 0) -> dict:
    """Small uniform-random sparse problem (edge-case tests): CSR with fp32 values in (-1, 1),
    labels y ~ N(0,1); the last ``empty_rows`` rows / ``empty_cols`` columns are empty."""
    rng = np.random.Generator(np.random.PCG64(seed))
    mask = rng.random((n_rows, n_cols)) < density
    if empty_rows:
        mask[n_rows - empty_rows:, :] = False
    if empty_cols:
        mask[:, n_cols - empty_cols:] = False
    vals = (rng.random((n_rows, n_cols)) * 2 - 1).astype(np.float32)
    ptr = np.zeros(n_rows + 1, np.int64)
    np.cumsum(mask.sum(1), out=ptr[1:])
    r, c = np.nonzero(mask)
    y = rng.standard_normal(n_rows).astype(np.float32)
    return dict(ptr=ptr, idx=c.astype(np.int32), val=vals[r, c].astype(np.float32), y=y, n_rows=n_rows,
                n_cols=n_cols, lam=1e-2, name=f"rand{n_rows}x{n_cols}")


# ----------------------------------------------------------------------------- device twin
def gen_device(cfg, row0: int = 0, nrows: int | None = None, stream=None) -> dict:
    """Generate rows [row0, row0+nrows) directly into CUDA memory (torch tensors)."""
    import torch

    nrows = cfg.n_rows - row0 if nrows is None else nrows
    lens = row_lengths(cfg, row0, nrows)
    nnz = int(lens.sum())
    dev = torch.device("cuda", torch.cuda.current_device())
    ptr = torch.empty(nrows + 1, dtype=torch.int64, device=dev)
    idx = torch.empty(max(nnz, 1), dtype=torch.int32, device=dev)
    val = torch.empty(max(nnz, 1), dtype=torch.float32, device=dev)
    y = torch.empty(max(nrows, 1), dtype=torch.float32, device=dev)
    s = stream if stream is not None else torch.cuda.current_stream()
    st, keep = cfg.struct()
    lib = _lib_cuda()
    if isinstance(cfg, FieldsCfg):
        rc = lib.synth_fields_fill_device(C.byref(st), row0, nrows, ptr.data_ptr(), idx.data_ptr(), val.data_ptr(),
                                          y.data_ptr(), C.c_void_p(s.cuda_stream))
    else:
        rc = lib.synth_zipf_fill_device(C.byref(st), row0, nrows, ptr.data_ptr(), idx.data_ptr(), val.data_ptr(),
                                        y.data_ptr(), C.c_void_p(s.cuda_stream))
    if rc:
        raise RuntimeError(f"synth device fill failed rc={rc}")
    s.synchronize()
    return dict(ptr=ptr, idx=idx[:nnz], val=val[:nnz], y=y[:nrows], n_rows=nrows, n_cols=cfg.n_cols,
                lam=cfg.lam, name=cfg.name)
