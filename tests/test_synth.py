"""Seeded input generators (synth/): invariants of the generated matrices and labels (CPU).
The device twin is checked bit-exact against the host twin in tests/test_gpu_parity.py."""
import numpy as np
import pytest

import synth


def _check_csr(d):
    ptr, idx = d["ptr"], d["idx"]
    assert ptr[0] == 0 and np.all(np.diff(ptr) >= 0) and ptr[-1] == len(idx)
    assert idx.min() >= 0 and idx.max() < d["n_cols"]
    for r in range(min(d["n_rows"], 300)):
        assert np.all(np.diff(idx[ptr[r]:ptr[r + 1]]) > 0)


def test_zipf_rows_invariants_and_shape():
    cfg = synth.CONFIGS["C2"].with_rows(3000)
    d = synth.gen_host(cfg)
    _check_csr(d)
    lens = np.diff(d["ptr"])
    assert 400 < lens.mean() < 600 and lens.min() >= 16 and lens.max() <= 5000
    assert np.all((d["val"] > 0) & (d["val"] <= 1))
    assert set(np.unique(d["y"]).tolist()) <= {-1.0, 1.0}
    # power-law column popularity: low ids (frequency ranks) far more common than high ids
    cnt = np.bincount(d["idx"], minlength=cfg.n_cols)
    assert cnt[:10].mean() > 20 * cnt[-10000:].mean()


def test_row_window_consistency_and_determinism():
    cfg = synth.CONFIGS["C3"].with_rows(400)
    a = synth.gen_host(cfg)
    b = synth.gen_host(cfg, row0=150, nrows=100)
    s, e = a["ptr"][150], a["ptr"][250]
    assert np.array_equal(b["idx"], a["idx"][s:e]) and np.array_equal(b["val"], a["val"][s:e])
    assert np.array_equal(b["y"], a["y"][150:250])
    c = synth.gen_host(cfg, threads=1)
    assert np.array_equal(c["idx"], a["idx"]) and np.array_equal(c["val"], a["val"])


def test_c3_row_lengths_match_recipe():
    cfg = synth.CONFIGS["C3"]
    lens = synth.row_lengths(cfg, 0, 200_000)
    assert 3600 < lens.mean() < 3850 and lens.min() >= 64 and lens.max() <= 16384
    t = synth.lognormal_len_table(3728.0, 0.6, 64, 16384)
    assert abs(t.mean() - 3728) < 2


def test_fields_generator():
    cfg = synth.c5_scaled(5000, 1e-3)
    d = synth.gen_host(cfg)
    _check_csr(d)
    nf = len(cfg.cards)
    assert np.all(np.diff(d["ptr"]) == nf) and np.all(d["val"] == 1.0)
    off = cfg.offsets
    fld = np.searchsorted(off, d["idx"], side="right") - 1
    assert np.array_equal(fld.reshape(-1, nf), np.tile(np.arange(nf), (5000, 1)))


def test_random_sparse_edge_rows():
    d = synth.random_sparse(20, 10, 0.5, 1, empty_rows=2, empty_cols=3)
    _check_csr(d)
    assert np.all(np.diff(d["ptr"])[-2:] == 0)
    assert not np.isin(np.arange(7, 10), d["idx"]).any()
