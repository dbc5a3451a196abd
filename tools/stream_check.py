"""Epoch time vs how the context's stream/memory were set up (diagnostic)."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth, paper_1702_07005_b200 as scd
cfg = synth.CONFIGS["C3"]; d = synth.gen_device(cfg)
mode = sys.argv[1]
def run(tag, stream=None):
    s = scd.Solver(d["ptr"], d["idx"], d["val"], d["n_rows"], d["n_cols"], d["y"], cfg.lam, "dual", seed=4, stream=stream)
    es = torch.cuda.ExternalStream(s.stream_handle)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.epoch(1); torch.cuda.synchronize()
    e0.record(es)
    for t in range(2, 6): s.epoch(t)
    e1.record(es); torch.cuda.synchronize()
    print(mode, tag, "%.2f ms/epoch" % (e0.elapsed_time(e1) / 4), flush=True)
    return s
if mode == "A": run("own")
if mode == "B": torch.cuda.Stream(); run("own-after-torch-stream")
if mode == "C": run("torch", torch.cuda.Stream())
if mode == "D": run("own").close(); run("own-second")
if mode == "E": s1 = run("own"); run("own-second-while-first-alive")
if mode == "F": x = torch.empty(256 << 20, dtype=torch.uint8, device="cuda"); run("own-after-256MB-alloc")
