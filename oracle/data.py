"""oracle.data — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): plain reference versions of the
data-layer utilities of the build (SURVEY L0 / K8'), written from their definitions, slow and
obviously correct.

``renumber``      the inner index space renumbered by frequency: new id = rank of the old index by
                  (number of stored entries, descending; index, ascending); entries relabelled and
                  re-sorted within each outer index.  ("renumbered by frequency at
                  load".)  Parity unpinned beyond its definition (no paper values): pinned by
                  invariants and a hand example (tests/golden/data_hand_values.json).
``parse_libsvm``  the LIBSVM text format the paper's datasets come in (webspam, criteo; P:254,
                  P:460): one example per line, ``label index:value ...`` with 1-based increasing
                  indices; returns CSR with 0-based indices (SPEC S:44-52 reading: blank lines and
                  ``#`` comments skipped, values parsed as float32).
"""
from __future__ import annotations

import numpy as np


def renumber(ptr, idx, val, n_inner: int):
    """Returns (ptr, idx, val, new_of_old) of the renumbered matrix (same outer layout)."""
    ptr = np.asarray(ptr, np.int64)
    idx = np.asarray(idx, np.int64)
    counts = np.bincount(idx, minlength=n_inner)
    order = sorted(range(n_inner), key=lambda j: (-int(counts[j]), j))  # rank r -> old index
    new_of_old = np.empty(n_inner, np.int32)
    for r, j in enumerate(order):
        new_of_old[j] = r
    out_idx = np.empty(len(idx), np.int32)
    out_val = None if val is None else np.empty(len(idx), np.float32)
    for o in range(len(ptr) - 1):
        b, e = int(ptr[o]), int(ptr[o + 1])
        pairs = sorted((int(new_of_old[idx[k]]), k) for k in range(b, e))
        for t, (nj, k) in enumerate(pairs):
            out_idx[b + t] = nj
            if val is not None:
                out_val[b + t] = val[k]
    return ptr.copy(), out_idx, out_val, new_of_old


def parse_libsvm(text: str, n_cols: int | None = None):
    """CSR dict(ptr, idx, val, y, n_rows, n_cols) of a LIBSVM-format text (0-based indices)."""
    ptr, idx, val, y = [0], [], [], []
    max_j = -1
    for line in text.splitlines():
        line = line.split("#", 1)[0].strip()
        if not line:
            continue
        parts = line.split()
        y.append(np.float32(float(parts[0])))
        last = -1
        for tok in parts[1:]:
            j_s, v_s = tok.split(":")
            j = int(j_s) - 1
            if j < 0 or j <= last:
                raise ValueError(f"bad index {j_s} (1-based, strictly increasing per line)")
            last = j
            idx.append(j)
            val.append(np.float32(float(v_s)))
            max_j = max(max_j, j)
        ptr.append(len(idx))
    nc = n_cols if n_cols is not None else max_j + 1
    if max_j >= nc:
        raise ValueError("index beyond n_cols")
    return dict(ptr=np.asarray(ptr, np.int64), idx=np.asarray(idx, np.int32), val=np.asarray(val, np.float32),
                y=np.asarray(y, np.float32), n_rows=len(y), n_cols=int(nc))
