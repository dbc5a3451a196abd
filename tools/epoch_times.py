"""Per-epoch device time over many epochs (does the epoch slow down as the model converges?)."""
import os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
import paper_1702_07005_b200 as scd
cfg = synth.CONFIGS[sys.argv[1]]
E = int(sys.argv[2])
d = synth.gen_device(cfg)
st = torch.cuda.Stream()
s = scd.Solver(d["ptr"], d["idx"], d["val"], d["n_rows"], d["n_cols"], d["y"], cfg.lam, "dual", seed=4, stream=st)
evs = [torch.cuda.Event(enable_timing=True) for _ in range(E + 1)]
evs[0].record(st)
for t in range(1, E + 1):
    s.epoch(t)
    evs[t].record(st)
torch.cuda.synchronize()
print("back-to-back ms:", " ".join("%.2f" % evs[i].elapsed_time(evs[i + 1]) for i in range(E)))
s.set_model(torch.zeros(d["n_rows"]).numpy())
ms = []
for t in range(1, E + 1):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st); s.epoch(t); e1.record(st); torch.cuda.synchronize(); ms.append(e0.elapsed_time(e1))
print("synced ms:      ", " ".join("%.2f" % m for m in ms))
x = s.get_model()
print("model |x| max %.3e" % abs(x).max())
