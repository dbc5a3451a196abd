"""Alg. 3/4 with K logical workers in the fp64 oracle (sequential local epochs) on a full-size
config: the reference trajectory (γ and gap per round) for the GPU's distributed runs.

  python tools/oracle_dist.py C4 2 optimal 25     # C3's matrix by feature, K = 2, optimal γ
  python tools/oracle_dist.py C5p 8 optimal 15 2000000   # criteo-shaped prefix by example

Output: one line per round and profiles/data/oracle_dist_<cfg>_K<k>_<mode>.json."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import synth
    from oracle import solver

    which, K, mode, rounds = sys.argv[1], int(sys.argv[2]), sys.argv[3], int(sys.argv[4])
    t0 = time.perf_counter()
    if which == "C4":
        d = synth.gen_host(synth.CONFIGS["C3"], threads=0)
        form, seed, seed_part, lam = "primal", 4, 4, 1e-3
    else:
        rows = int(sys.argv[5]) if len(sys.argv) > 5 else 2_000_000
        d = synth.gen_host(synth.CONFIGS["C5"].with_rows(rows), threads=0)
        form, seed, seed_part, lam = "dual", 5, 5, 1e-3 * 200_000_000 / rows  # λN = 2e5 as in C5
    pr = solver.Problem.from_csr(d, lam=lam)
    del d
    print(f"setup {time.perf_counter() - t0:.1f} s", flush=True)
    t0 = time.perf_counter()
    _, _, hist = solver.run_distributed(pr, form, K, mode, rounds, seed=seed, seed_part=seed_part)
    el = time.perf_counter() - t0
    for h in hist:
        print(f"round {h['epoch']}: gamma {h['gamma']:.4f} gap {h['gap']:.3e} P {h['P']:.12g}", flush=True)
    print(f"{rounds} rounds in {el:.1f} s (incl. evaluation)")
    os.makedirs(os.path.join(ROOT, "profiles", "data"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", "data", f"oracle_dist_{which}_K{K}_{mode}.json"), "w") as f:
        json.dump(dict(config=which, K=K, mode=mode, rounds=rounds, seconds=el, hist=hist), f, indent=1)


if __name__ == "__main__":
    main()
