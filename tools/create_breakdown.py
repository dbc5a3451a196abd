"""Where does scd_create from host buffers spend its time (the e2e step of bench.py)?
Times: the raw pinned H2D copy of the same arrays (torch), scd_create with the default setup,
with the placement probe disabled (SCD_SV_TUNE=0), and the epoch time with each placement.
Usage: python tools/create_breakdown.py C3"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_1702_07005_b200 as scd  # noqa: E402

cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C3"]
d = synth.gen_device(cfg)
rows, nnz = d["n_rows"], d["idx"].numel()
hp = torch.empty(rows + 1, dtype=torch.int64, pin_memory=True).copy_(d["ptr"])
hi = torch.empty(nnz, dtype=torch.int32, pin_memory=True).copy_(d["idx"])
hv = torch.empty(nnz, dtype=torch.float32, pin_memory=True).copy_(d["val"])
hy = torch.empty(rows, dtype=torch.float32, pin_memory=True).copy_(d["y"])
del d
torch.cuda.empty_cache()
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    g = [x.cuda(non_blocking=True) for x in (hp, hi, hv, hy)]
    torch.cuda.synchronize()
    print(f"raw H2D {sum(x.numel() * x.element_size() for x in g) / 1e9:.2f} GB: {time.perf_counter() - t0:.3f} s",
          flush=True)
    del g
    torch.cuda.empty_cache()
for tune in ("1", "0"):
    os.environ["SCD_SV_TUNE"] = tune
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        s = scd.Solver(hp, hi, hv, rows, cfg.n_cols, hy, cfg.lam, "dual", seed=3, validate=False)
        t1 = time.perf_counter()
        es = torch.cuda.ExternalStream(s.stream_handle)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.epoch(1)
        e0.record(es)
        for t in range(2, 6):
            s.epoch(t)
        e1.record(es)
        torch.cuda.synchronize()
        inf = s.info()
        print(f"tune={tune}: create {t1 - t0:.3f} s, offset {inf['sv_offset_bytes']}, probe {inf['probe_ms']}, "
              f"epoch {e0.elapsed_time(e1) / 4:.2f} ms", flush=True)
        s.close()
# device-resident inputs: the create-time analysis alone (validation, norms, schedule, staleness
# estimates, placement probe), with and without the tail-copy estimate and the probe
dp, di, dv, dy = (x.cuda() for x in (hp, hi, hv, hy))
for env in ({}, {"SCD_TAIL_SNAP": "0"}, {"SCD_SV_TUNE": "0"}, {"SCD_TAIL_SNAP": "0", "SCD_SV_TUNE": "0"}):
    for k in ("SCD_TAIL_SNAP", "SCD_SV_TUNE"):
        os.environ.pop(k, None)
    os.environ.update(env)
    ts = []
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        s = scd.Solver(dp, di, dv, rows, cfg.n_cols, dy, cfg.lam, "dual", seed=3)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
        s.close()
    print(f"device inputs {env or 'default'}: create " + " ".join(f"{t:.3f}" for t in ts) + " s", flush=True)
