"""Epoch time vs the byte offset of the shared vector inside its allocation (diagnostic)."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth, paper_1702_07005_b200 as scd
cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C3"]; d = synth.gen_device(cfg)
for off in [int(x) for x in os.environ.get("OFFS", "0,4096").split(",")]:
    os.environ["SCD_SV_OFFSET"] = str(off)
    s = scd.Solver(d["ptr"], d["idx"], d["val"], d["n_rows"], d["n_cols"], d["y"], cfg.lam, "dual", seed=4)
    es = torch.cuda.ExternalStream(s.stream_handle)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.epoch(1); torch.cuda.synchronize()
    e0.record(es)
    for t in range(2, 5): s.epoch(t)
    e1.record(es); torch.cuda.synchronize()
    print("offset %8d: %.2f ms/epoch" % (off, e0.elapsed_time(e1) / 3), flush=True)
    s.close()
