"""C-ABI library loads and exports every symbol include/scd.h declares (CPU, no compute calls);
argument validation that happens before any CUDA call; the oracle/product separation."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "scd.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(scd_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    import paper_1702_07005_b200 as p

    lib = p.lib()
    names = _declared()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), f"libscd.so does not export {n}"
    assert set(names) == set(p.scd.EXPORTS)


def test_invalid_arguments_rejected_before_any_device_work():
    import paper_1702_07005_b200 as p
    from paper_1702_07005_b200.scd import ScdError

    ptr = np.array([0, 1], np.int64)
    idx = np.array([0], np.int32)
    val = np.array([1.0], np.float32)
    y = np.array([1.0], np.float32)
    for lam in (0.0, -1.0, float("nan")):
        with pytest.raises(ScdError) as e:
            p.Solver(ptr, idx, val, 1, 1, y, lam, "dual")
        assert e.value.status == 1  # SCD_E_INVALID_ARG
    with pytest.raises(ScdError) as e:  # world > 1 without a communicator
        p.Solver(ptr, idx, val, 1, 1, y, 1.0, "dual", world=2, rank=0)
    assert e.value.status == 6  # SCD_E_STATE
    with pytest.raises(ScdError) as e:
        p.Solver(ptr, idx, val, 0, 1, y, 1.0, "dual")
    assert e.value.status == 1


def test_binding_structs_match_the_header():
    """The ctypes mirrors of scd_matrix / scd_options / scd_info have the C sizes (a field added to
    the header but not to the binding would corrupt memory)."""
    import paper_1702_07005_b200 as p
    from paper_1702_07005_b200 import scd as b

    out = (ctypes.c_int64 * 4)()
    p.lib().scd_struct_sizes(out)
    assert list(out) == [ctypes.sizeof(b.Matrix), ctypes.sizeof(b.Options), ctypes.sizeof(b.Info),
                         ctypes.sizeof(b.Collectives)]


def test_status_strings():
    import paper_1702_07005_b200 as p

    lib = p.lib()
    assert lib.scd_status_string(2) == b"SCD_E_BAD_MATRIX"


def test_product_does_not_import_or_link_oracle():
    """The CUDA product path shares no code with the oracle (and never falls back to it)."""
    pkg = os.path.join(ROOT, "paper_1702_07005_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "import synth" not in txt, f
    so = open(os.path.join(pkg, "libscd.so"), "rb").read()
    assert b"orc_" not in so and b"liboracle" not in so
