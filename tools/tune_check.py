"""Placement probe check: chosen offset, probe spread, and the real epoch time per context."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth, paper_1702_07005_b200 as scd
cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C3"]; d = synth.gen_device(cfg)
for rep in range(int(sys.argv[2]) if len(sys.argv) > 2 else 3):
    if rep == 1: torch.cuda.Stream()  # perturb allocations like the bench did
    s = scd.Solver(d["ptr"], d["idx"], d["val"], d["n_rows"], d["n_cols"], d["y"], cfg.lam, "dual", seed=4)
    inf = s.info()
    es = torch.cuda.ExternalStream(s.stream_handle)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.epoch(1); torch.cuda.synchronize()
    e0.record(es)
    for t in range(2, 5): s.epoch(t)
    e1.record(es); torch.cuda.synchronize()
    print("rep %d offset %6d probe best/worst %.3f/%.3f ms -> epoch %.2f ms" % (rep, inf["sv_offset_bytes"], *inf["probe_ms"], e0.elapsed_time(e1) / 3), flush=True)
