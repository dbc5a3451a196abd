"""Summaries for profiles/ (run here, on the CPU box, on files gpurun brought back).

  python tools/summarize_profiles.py launches gpurun_out/launches.csv [last [skip_tail]] > profiles/launches_r1.md
  python tools/summarize_profiles.py ncu gpurun_out/prof.ncu-rep profiles/ncu_epoch_r1  [bytes_per_launch]

`launches`: per-kernel launch count, total and mean device time, share of the listed time
(ncu --metrics gpu__time_duration.sum --clock-control none; cold-cache and serialised, so
compare shares, not absolutes).
`ncu`: key metrics of one --set full capture (duration, DRAM bytes, L2/L1 throughput, occupancy,
stall reasons) as markdown + JSON; writes profiles/ncu_traffic.json (dram bytes per launch).
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict


def launches(path, last=0, skip=0):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi, mi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    agg = defaultdict(lambda: [0, 0.0])
    body = rows[1:]
    if skip:
        body = body[:-skip]
    if last:
        body = body[-last:]
        print(f"Last {last} launches of the list" + (f" before the final {skip}" if skip else "") +
              " (the timed region).\n")
    for r in body:
        if r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0].replace("<unnamed>::", "").replace("scd::", "")
        agg[name][0] += 1
        agg[name][1] += float(r[vi].replace(",", "")) / 1e6
    tot = sum(v[1] for v in agg.values())
    print(f"| kernel | launches | total ms | mean ms | share |\n|---|---|---|---|---|")
    for k, (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| `{k[:90]}` | {n} | {ms:.3f} | {ms / n:.4f} | {100 * ms / tot:.1f}% |")
    print(f"\nTotal listed device time: {tot:.3f} ms")


KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_tag_requests.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_requests.sum", "lts__t_sectors_srcunit_tex_op_red.sum", "lts__t_sectors_srcunit_tex_op_read.sum",
    "lts__t_sectors_srcunit_ltcfabric.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "smsp__inst_executed_op_global_red.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
]


def ncu(rep, out_prefix, bytes_per_launch=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {h: (v, u) for h, u, v in zip(hdr, units, vals)}
        m = {k: d[k] for k in KEYS if k in d}
        st = sorted([(h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""),
                      float(v)) for h, (v, u) in d.items()
                     if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")
                     and v not in ("", "n/a")], key=lambda x: -x[1])[:6]
        res.append(dict(kernel=d.get("Kernel Name", ("?", ""))[0], metrics=m, stalls=st))
    md = [f"# ncu --set full summary: `{os.path.basename(rep)}`\n"]
    js = []
    for r in res:
        md.append(f"## `{r['kernel'][:120]}`\n\n| metric | value | unit |\n|---|---|---|")
        for k, (v, u) in r["metrics"].items():
            md.append(f"| {k} | {v} | {u} |")
        md.append("\nTop warp stall reasons (cycles per issued instruction): " +
                  ", ".join(f"{a} {b:.1f}" for a, b in r["stalls"]) + "\n")
        rd = r["metrics"].get("dram__bytes_read.sum")
        wr = r["metrics"].get("dram__bytes_write.sum")

        def tobytes(x):
            if not x:
                return None
            v, u = x
            v = float(v.replace(",", ""))
            return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)

        traffic = (tobytes(rd) or 0) + (tobytes(wr) or 0)
        l2 = r["metrics"].get("lts__t_tag_requests.avg.pct_of_peak_sustained_elapsed")
        js.append(dict(kernel=r["kernel"], dram_bytes_per_launch=traffic,
                       duration=r["metrics"].get("gpu__time_duration.sum"),
                       l2_tag_requests_pct=float(l2[0].replace(",", "")) if l2 else None))
        if bytes_per_launch:
            md.append(f"Algorithmic bytes per launch (16 B/nnz + 32 B/coord model): {bytes_per_launch:.4g}; "
                      f"measured DRAM traffic per launch: {traffic:.4g} B ({traffic / bytes_per_launch:.2f}x).\n")
    open(out_prefix + ".md", "w").write("\n".join(md))
    json.dump(js, open(out_prefix + ".json", "w"), indent=1)
    if js:
        # per-kernel map (short name -> DRAM bytes per launch of the last capture), read by bench.py
        tp = os.path.join(os.path.dirname(out_prefix), "ncu_traffic.json")
        try:
            cur = json.load(open(tp))
        except Exception:
            cur = {}
        if "kernel" in cur:  # old single-kernel format
            cur = {}
        for r in js:
            short = r["kernel"].split("<")[0].split("::")[-1].replace("void ", "").strip()
            cur[short] = dict(source=os.path.basename(out_prefix) + ".json", kernel=r["kernel"],
                              dram_bytes_per_launch=r["dram_bytes_per_launch"],
                              l2_tag_requests_pct=r.get("l2_tag_requests_pct"))
        json.dump(cur, open(tp, "w"), indent=1)
    print("\n".join(md))


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 0, int(sys.argv[4]) if len(sys.argv) > 4 else 0)
    else:
        ncu(sys.argv[2], sys.argv[3], float(sys.argv[4]) if len(sys.argv) > 4 else None)
