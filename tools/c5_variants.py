"""C5 shard (25 M rows, implicit values, global N = 200 M as in the 8-GPU run): epoch time and per-epoch
gap of schedule variants (each in its own process; env knobs are read at create).

  python tools/c5_variants.py 4 "" "SCD_BLOCK=32"
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def child(E):
    import torch

    import synth
    import paper_1702_07005_b200 as scd

    cfg = synth.CONFIGS["C5"]
    d = synth.gen_device(cfg, 0, 25_000_000)
    s = scd.Solver(d["ptr"], d["idx"], None, 25_000_000, cfg.n_cols, d["y"], cfg.lam, "dual", seed=5,
                   n_global=cfg.n_rows)
    st = torch.cuda.ExternalStream(s.stream_handle)
    rows = []
    for t in range(1, E + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        s.epoch(t)
        e1.record(st)
        torch.cuda.synchronize()
        rows.append((e0.elapsed_time(e1), s.duality_gap()))
    info = s.info()
    s.close()
    print("RESULT " + json.dumps(dict(rows=rows, bins=info["bins"], hot_copy=info["hot_copy"], hot_tp=info["hot_tp"])))


def main():
    if sys.argv[1] == "--child":
        return child(int(sys.argv[2]))
    E = int(sys.argv[1])
    for var in sys.argv[2:]:
        env = dict(os.environ)
        for kv in var.split():
            k, v = kv.split("=")
            env[k] = v
        r = subprocess.run([sys.executable, __file__, "--child", str(E)], env=env, capture_output=True, text=True)
        line = [x for x in r.stdout.splitlines() if x.startswith("RESULT ")]
        if not line:
            print(var or "(default)", "FAILED", r.stderr[-800:])
            continue
        res = json.loads(line[0][7:])
        ms = sorted(x[0] for x in res["rows"])[len(res["rows"]) // 2]
        b = res["bins"][0]
        print(f"{var or '(default)':32s} {ms:7.2f} ms/epoch  gaps " + " ".join(f"{g:.2e}" for _, g in res["rows"]) +
              f"  grid {b['grid']} F {b['flush']} hot {b['hot']} copy {res['hot_copy']} tp {res['hot_tp']}", flush=True)


if __name__ == "__main__":
    main()
