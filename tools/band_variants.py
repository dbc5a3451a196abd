"""GPU-only per-epoch gaps of schedule variants at full size, compared with a recorded oracle run
(tools/fullsize_band.py output).  Each variant runs in its own process (env knobs are read at create).

  python tools/band_variants.py C4 6 "" "SCD_SLICES=16" "BV_MAXIN=32" "BV_DET=1"
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def child(which, E):
    import torch

    import synth
    import paper_1702_07005_b200 as scd

    cfg = synth.CONFIGS["C3"]
    d = synth.gen_device(cfg)
    N, M = d["n_rows"], d["n_cols"]
    if which == "C3":
        s = scd.Solver(d["ptr"], d["idx"], d["val"], N, M, d["y"], cfg.lam, "dual", seed=3)
    else:
        cp, ci, cv = scd.transpose(d["ptr"], d["idx"], d["val"], N, M, "csr")
        s = scd.Solver(cp, ci, cv, N, M, d["y"], cfg.lam, "primal", seed=4,
                       deterministic=os.environ.get("BV_DET") == "1", max_inflight=int(os.environ.get("BV_MAXIN", "0")))
    st = torch.cuda.ExternalStream(s.stream_handle)
    out = []
    for t in range(1, E + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        s.epoch(t)
        e1.record(st)
        torch.cuda.synchronize()
        out.append((e0.elapsed_time(e1), s.duality_gap()))
    info = s.info()
    s.close()
    print("RESULT " + json.dumps(dict(rows=out, bins=info["bins"], n_slices=info["n_slices"],
                                      sm={k: info.get(k) for k in ("sm_head", "sm_ch", "sm_rh", "tail_roll", "head_copy")})))


def main():
    if sys.argv[1] == "--child":
        return child(sys.argv[2], int(sys.argv[3]))
    which, E = sys.argv[1], int(sys.argv[2])
    ref = json.load(open(os.path.join(ROOT, "profiles", "data", f"band_{which}.json")))
    orc = [o["gap"] for o in ref["oracle"]]
    for var in sys.argv[3:]:
        env = dict(os.environ)
        for kv in var.split():
            k, v = kv.split("=")
            env[k] = v
        r = subprocess.run([sys.executable, __file__, "--child", which, str(E)], env=env, capture_output=True, text=True)
        line = [x for x in r.stdout.splitlines() if x.startswith("RESULT ")]
        if not line:
            print(var or "(default)", "FAILED", r.stderr[-800:])
            continue
        res = json.loads(line[0][7:])
        ms = sum(x[0] for x in res["rows"][1:]) / max(1, len(res["rows"]) - 1)
        ratios = " ".join(f"{g / o:.2f}" for (_, g), o in zip(res["rows"], orc))
        gaps = " ".join(f"{g:.2e}" for _, g in res["rows"])
        print(f"{var or '(default)':40s} {ms:7.2f} ms/epoch  gaps {gaps}  ratio {ratios}  {res.get('sm')}", flush=True)


if __name__ == "__main__":
    main()
