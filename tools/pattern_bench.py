"""Access-pattern ceiling of the epoch (tools/pattern_bench.cu) on a config's own matrix:
stream only / + gathers / + reds / both, over all stored entries in storage order.
Usage: python tools/pattern_bench.py C3 [rows]"""
import ctypes as C
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402

lib = C.CDLL(os.path.join(ROOT, "tools", "libpattern.so"))
lib.pattern_run.restype = C.c_float
lib.pattern_run.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]
name = sys.argv[1]
cfg = synth.CONFIGS["C5"].with_rows(int(sys.argv[2])) if name == "C5" else synth.CONFIGS[name]
d = synth.gen_device(cfg)
nnz = d["idx"].numel()
sv = torch.zeros(cfg.n_cols + 65536, device="cuda")
sink = torch.zeros(1, device="cuda")
for off in (0, 1024):  # two placements of the vector
    for mode, nm in ((0, "stream idx+val"), (1, "+ gather"), (2, "+ red"), (3, "+ gather + red")):
        ms = min(lib.pattern_run(mode, d["idx"].data_ptr(), d["val"].data_ptr(), nnz, sv[off:].data_ptr(),
                                 sink.data_ptr()) for _ in range(3))
        print(f"{name} off={off * 4:6d}B {nm:16s}: {ms:7.3f} ms  {nnz / ms / 1e6:7.1f} G entries/s", flush=True)
