"""Data-layer utilities (SURVEY L0 / K8'): the oracle's frequency renumbering and LIBSVM parser
pinned to hand values and invariants (CPU), the C-ABI versions bit-exact against them (GPU)."""
import json
import os

import numpy as np
import pytest

import synth
from oracle import data as odata

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def golden():
    return json.load(open(os.path.join(HERE, "golden", "data_hand_values.json")))


def test_renumber_hand_example(golden):
    g = golden["renumber"]
    p, i, v, m = odata.renumber(np.array(g["ptr"]), np.array(g["idx"]), np.array(g["val"], np.float32), g["n_inner"])
    assert p.tolist() == g["ptr"] and i.tolist() == g["out_idx"] and m.tolist() == g["new_of_old"]
    assert np.allclose(v, g["out_val"])


def _check_renumber_invariants(ptr, idx, val, n_inner, out):
    p, i, v, m = out
    assert np.array_equal(p, ptr)
    assert np.array_equal(np.sort(m), np.arange(n_inner))  # a bijection
    counts_old = np.bincount(idx, minlength=n_inner)
    counts_new = np.bincount(i, minlength=n_inner)
    assert np.array_equal(counts_new[m], counts_old)          # entries follow their index
    assert np.all(np.diff(counts_new) <= 0)                   # frequency-ranked
    ties = np.nonzero(np.diff(counts_new) == 0)[0]            # equal counts keep the old order
    inv = np.argsort(m)
    assert np.all(inv[ties] < inv[ties + 1])
    for o in range(len(ptr) - 1):
        b, e = ptr[o], ptr[o + 1]
        assert np.all(np.diff(i[b:e]) > 0)                    # sorted within each outer index
        got = sorted(zip(inv[i[b:e]].tolist(), v[b:e].tolist()))
        ref = sorted(zip(idx[b:e].tolist(), val[b:e].tolist()))
        assert got == ref                                     # same (old index, value) pairs


def test_renumber_invariants_random_with_empty_rows_and_columns():
    d = synth.random_sparse(120, 60, 0.08, 5, empty_rows=4, empty_cols=6)
    out = odata.renumber(d["ptr"], d["idx"], d["val"], 60)
    _check_renumber_invariants(d["ptr"], d["idx"], d["val"], 60, out)


def test_libsvm_hand_example(golden):
    g = golden["libsvm"]
    d = odata.parse_libsvm(g["text"])
    assert d["ptr"].tolist() == g["ptr"] and d["idx"].tolist() == g["idx"] and d["n_cols"] == g["n_cols"]
    assert np.array_equal(d["val"], np.array(g["val"], np.float32))
    assert np.array_equal(d["y"], np.array(g["y"], np.float32))
    with pytest.raises(ValueError):
        odata.parse_libsvm("1 3:1 2:1\n")  # decreasing indices


def test_libsvm_library_reader_matches_oracle(tmp_path, golden):
    """The library's LIBSVM reader (scd_load_libsvm, host C++) — bit-exact with the oracle parser on
    the hand example and on a synthetic file written from a C2 prefix (%.9g round-trips fp32)."""
    import paper_1702_07005_b200 as scd

    f = tmp_path / "hand.svm"
    f.write_text(golden["libsvm"]["text"])
    got = scd.load_libsvm(str(f))
    ref = odata.parse_libsvm(golden["libsvm"]["text"])
    for k in ("ptr", "idx", "val", "y"):
        assert np.array_equal(got[k], ref[k]), k
    assert got["n_rows"] == ref["n_rows"] and got["n_cols"] == ref["n_cols"]
    d = synth.gen_host(synth.CONFIGS["C2"].with_rows(300))
    lines = []
    for r in range(300):
        b, e = d["ptr"][r], d["ptr"][r + 1]
        feats = " ".join(f"{j + 1}:{v:.9g}" for j, v in zip(d["idx"][b:e], d["val"][b:e]))
        lines.append(f"{d['y'][r]:.9g} {feats}")
    f2 = tmp_path / "c2.svm"
    f2.write_text("\n".join(lines) + "\n")
    got = scd.load_libsvm(str(f2), n_cols=d["n_cols"])
    for k in ("ptr", "idx", "val", "y"):
        assert np.array_equal(got[k], d[k]), k
    ref = odata.parse_libsvm(f2.read_text(), n_cols=d["n_cols"])
    for k in ("ptr", "idx", "val", "y"):
        assert np.array_equal(got[k], ref[k]), k
    bad = tmp_path / "bad.svm"
    bad.write_text("1 3:1 2:1\n")
    with pytest.raises(Exception):
        scd.load_libsvm(str(bad))


@pytest.mark.gpu
@pytest.mark.parametrize("layout", ["csr", "csc"])
def test_renumber_device_bit_exact(layout):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():  # pragma: no cover
        pytest.skip("no CUDA device")
    import paper_1702_07005_b200 as scd

    d = synth.random_sparse(400, 150, 0.05, 11, empty_rows=5, empty_cols=9)
    ptr, idx, val = d["ptr"], d["idx"], d["val"]
    n_inner = 150
    if layout == "csc":
        ptr, idx, val = scd.transpose(ptr, idx, val, 400, 150, "csr")
        n_inner = 400
    ref = odata.renumber(ptr, idx, val, n_inner)
    got = scd.renumber(ptr, idx, val, 400, 150, layout)
    for a, b in zip(got, ref):
        assert np.array_equal(a, b)
    dev = [torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in (ptr, idx, val)]
    got = scd.renumber(*dev, 400, 150, layout)
    for a, b in zip(got, ref):
        assert np.array_equal(a.cpu().numpy(), b)
    # implicit values: pattern only
    gi = scd.renumber(ptr, idx, None, 400, 150, layout)
    assert gi[2] is None and np.array_equal(gi[1], ref[1]) and np.array_equal(gi[3], ref[3])


@pytest.mark.gpu
def test_renumber_c2_prefix_bit_exact_and_head_kernel_applies():
    """A C2 prefix with its columns scrambled by a random bijection: renumbering restores a
    frequency-ranked index space (the head of w̄ dense again), bit-exact with the oracle."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():  # pragma: no cover
        pytest.skip("no CUDA device")
    import paper_1702_07005_b200 as scd

    d = synth.gen_host(synth.CONFIGS["C2"].with_rows(2000))
    M = d["n_cols"]
    scramble = np.random.default_rng(0).permutation(M).astype(np.int32)
    idx = scramble[d["idx"]]
    p2, i2, v2 = [], [], []
    for r in range(2000):
        b, e = d["ptr"][r], d["ptr"][r + 1]
        o = np.argsort(idx[b:e])
        i2.append(idx[b:e][o])
        v2.append(d["val"][b:e][o])
    idx_s, val_s = np.concatenate(i2).astype(np.int32), np.concatenate(v2).astype(np.float32)
    ref = odata.renumber(d["ptr"], idx_s, val_s, M)
    got = scd.renumber(d["ptr"], idx_s, val_s, 2000, M, "csr")
    for a, b in zip(got, ref):
        assert np.array_equal(a, b)
    head = np.mean(got[1] < 8192)
    assert head > 0.5, head  # the frequency head is dense again (C2: Zipf over 50 000 features)
