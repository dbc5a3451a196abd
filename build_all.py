"""Native build for the repo (used by __graft_entry__.build() and tests/conftest.py).

Builds, in-tree, only when a source is newer than its target:
  paper_1702_07005_b200/libscd.so   product C-ABI library (nvcc, sm_100a, links NCCL)
  synth/libsynth_host.so            seeded input generator, host twin (gcc, OpenMP)
  synth/libsynth_cuda.so            seeded input generator, device twin (nvcc, sm_100a)
  oracle/liboracle.so               fp64 oracle (gcc) — test infrastructure, never linked by the product
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dirs():
    import nvidia.nccl as nc  # torch-bundled NCCL 2.28 (headers + libnccl.so.2)

    base = os.path.dirname(nc.__file__) if getattr(nc, "__file__", None) else list(nc.__path__)[0]
    return os.path.join(base, "include"), os.path.join(base, "lib")


def _stale(target: str, sources: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def _run(cmd: list[str], verbose: bool):
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"build failed: {' '.join(cmd[:3])} ...")
    if verbose and (r.stdout or r.stderr):
        print(r.stdout + r.stderr)


def nvcc() -> str:
    for c in ("/usr/local/cuda/bin/nvcc", "nvcc"):
        if os.path.exists(c) or c == "nvcc":
            return c
    return "nvcc"


def build_product(verbose=False, force=False):
    src = sorted(glob.glob(os.path.join(ROOT, "paper_1702_07005_b200/csrc/*.cu")))
    hdr = sorted(glob.glob(os.path.join(ROOT, "paper_1702_07005_b200/csrc/*.cuh"))) + \
        sorted(glob.glob(os.path.join(ROOT, "include/*.h")))
    out = os.path.join(ROOT, "paper_1702_07005_b200/libscd.so")
    if not src:
        return None
    if not force and not _stale(out, src + hdr):
        return out
    inc, lib = _nccl_dirs()
    cmd = [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC",
           "-Xptxas", "-v" if verbose else "-O3", "--expt-relaxed-constexpr",
           "-I", os.path.join(ROOT, "include"), "-I", inc, *src, "-o", out,
           "-L", lib, "-l:libnccl.so.2", f"-Xlinker=-rpath={lib}"]
    _run(cmd, verbose)
    return out


def build_synth(verbose=False, force=False):
    d = os.path.join(ROOT, "synth")
    h = os.path.join(d, "synth.h")
    out_h = os.path.join(d, "libsynth_host.so")
    if force or _stale(out_h, [os.path.join(d, "synth_host.c"), h]):
        _run(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-fopenmp", "-ffp-contract=off",
              os.path.join(d, "synth_host.c"), "-o", out_h, "-lm"], verbose)
    out_c = os.path.join(d, "libsynth_cuda.so")
    if force or _stale(out_c, [os.path.join(d, "synth_cuda.cu"), h]):
        _run([nvcc(), *ARCH, "-O3", "-std=c++17", "-shared", "-Xcompiler", "-fPIC", "-fmad=false",
              os.path.join(d, "synth_cuda.cu"), "-o", out_c], verbose)
    return out_h, out_c


def build_oracle(verbose=False, force=False):
    d = os.path.join(ROOT, "oracle")
    out = os.path.join(d, "liboracle.so")
    src = [os.path.join(d, "oracle.c")]
    if force or _stale(out, src):
        _run(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-ffp-contract=off", *src, "-o", out, "-lm"], verbose)
    return out


def build_tools(verbose=False, force=False):
    """Measurement tools used by bench.py (the access-pattern ceiling kernel)."""
    src = os.path.join(ROOT, "tools", "pattern_bench.cu")
    out = os.path.join(ROOT, "tools", "libpattern.so")
    if os.path.exists(src) and (force or _stale(out, [src])):
        _run([nvcc(), *ARCH, "-O3", "-std=c++17", "-shared", "-Xcompiler", "-fPIC", src, "-o", out], verbose)


def build(verbose=False, force=False, product=True):
    build_oracle(verbose, force)
    build_synth(verbose, force)
    if product:
        build_product(verbose, force)
        build_tools(verbose, force)


if __name__ == "__main__":
    build(verbose="-v" in sys.argv, force="-f" in sys.argv, product="--no-product" not in sys.argv)
