"""Access pattern of the C3 epoch split by home die (tools/die_pattern.cu): gather / RED / both over
all stored entries (storage order) with every SM on every entry, vs each die's SMs on the entries
homed on their own die (local) or on the other die (remote).  Usage: python tools/die_pattern.py C3"""
import ctypes as C
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402

lib = C.CDLL(os.path.join(ROOT, "tools", "libdiepattern.so"))
lib.die_map.restype = C.c_int
lib.die_map.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]
lib.die_pattern_run.restype = C.c_float
lib.die_pattern_run.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                                C.c_int, C.c_int, C.c_void_p]
cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C3"]
if len(sys.argv) > 2:
    cfg = cfg.with_rows(int(sys.argv[2]))
d = synth.gen_device(cfg)
idx = d["idx"]
nnz = idx.numel()
n = cfg.n_cols
sv = torch.zeros(n + 1024, device="cuda")
chunk_die = torch.zeros((n + 511) // 512, dtype=torch.uint8, device="cuda")
sm_die = torch.zeros(256, dtype=torch.uint8, device="cuda")
n0 = lib.die_map(sv.data_ptr(), n, chunk_die.data_ptr(), sm_die.data_ptr())
nsm = torch.cuda.get_device_properties(0).multi_processor_count
die_of = chunk_die[(idx // 512).long()]
l0 = idx[die_of == 0].contiguous()
l1 = idx[die_of == 1].contiguous()
print(f"SMs die0/die1 = {n0}/{nsm - n0}; entries die0 {l0.numel() / nnz:.3f}", flush=True)
sink = torch.zeros(1, device="cuda")
for mode, nm in ((1, "gather"), (2, "red"), (3, "gather+red")):
    for sel, sn in ((0, "all"), (1, "local"), (2, "remote")):
        a0, a1 = (idx, idx) if sel == 0 else (l0, l1)
        m0, m1 = (nnz, 0) if sel == 0 else (l0.numel(), l1.numel())
        ms = min(lib.die_pattern_run(mode, sel, a0.data_ptr(), m0, a1.data_ptr(), m1, sv.data_ptr(),
                                     sm_die.data_ptr(), n0, nsm - n0, sink.data_ptr()) for _ in range(3))
        print(f"{nm:11s} {sn:7s}: {ms:7.3f} ms  {nnz / ms / 1e6:7.1f} G entries/s", flush=True)
