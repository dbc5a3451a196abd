"""CPU: bench.py's reference arm (the fp64 oracle on a bounded sample of the C3 workload, timed on
the host cores) prints the contract's JSON line without a GPU."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "1"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = [x for x in r.stdout.splitlines() if x.startswith("{")][-1]
    d = json.loads(line)
    assert d["impl"] == "reference" and d["n_gpus"] == 1 and d["steps"] == 1 and d["warmup"] == 1
    assert d["metric"] == "nnz/s per epoch" and d["unit"] == "nnz/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["unit"] == d["unit"]
    assert d["config"]["workload"].startswith("C3 webspam-shaped")


@pytest.mark.gpu
def test_gpu_bench_json_line():
    """GPU: bench.py's own arm prints the contract's line: headline C3 metric, roofline of the dominant
    kernel (frac = achieved / peak), clocks sampled during the timed region, library launches counted,
    and the sub-records (C4 primal, C5 shard, the data layer's renumbering at full scale)."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "3", "--warmup", "3", "--quick",
                        "--no-cpu-baseline", "--no-e2e"], capture_output=True, text=True, timeout=1200, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
    assert d["metric"] == "nnz/s per epoch" and d["value"] > 0 and d["n_gpus"] == 1 and d["steps"] == 3
    assert d["config"]["nnz_per_gpu"] == 1306002649 and d["dtype"] == "f32"
    roof = d["roofline"]
    assert roof["kernel"].startswith("k_epoch_sm_tma") and abs(roof["frac"] - roof["achieved"] / roof["peak"]) < 1e-9
    assert 0.9 < roof["kernel_share_of_step"] <= 1.0
    assert d["clocks"]["samples"] >= 1 and d["gpu_launches"] == 2 * 3
    assert d["time_to_gap"]["gap_trace"][-1] <= 1e-4
    assert d["c4_primal"]["ms_per_step"] > 0 and d["c5_shard"]["ms_per_step"] > 0
    assert all(d["c3_load"]["checks"].values()), d["c3_load"]
    assert d["c2"]["dual"]["ms_per_step"] > 0 and d["c2"]["primal"]["time_to_gap"]["gap_trace"][-1] <= 1e-4
