#!/usr/bin/env python
"""Summarise ncu outputs into profiles/ (committed evidence).

    python tools/ncu_summary.py --launches gpurun_out/launches.csv \
        --full gpurun_out/bench_full.ncu-rep --out profiles/r01
Writes <out>_launches.md (per-kernel launch durations and shares) and
<out>_full.md + profiles/ncu_traffic.json (DRAM bytes / duration / key
metrics of the captured launches).
"""
import argparse
import csv
import io
import json
import os
import subprocess
from collections import defaultdict


def launches(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    per = defaultdict(list)
    for r in rows[start + 1:]:
        if len(r) <= iv:
            continue
        v = float(r[iv].replace(",", ""))
        unit = r[iu]
        us = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}[unit] * v
        per[r[ik]].append(us)
    return per


def full(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "dram__bytes_read.sum.pct_of_peak_sustained_elapsed", "dram__bytes_write.sum.pct_of_peak_sustained_elapsed",
            "dram__bytes.sum.per_second", "dram__bytes.sum.peak_sustained", "dram__cycles_elapsed.avg.per_second",
            "dram__cycles_active.avg.pct_of_peak_sustained_elapsed",
            "gpu__compute_memory_access_throughput.avg.pct_of_peak_sustained_elapsed",
            "launch__occupancy_limit_registers", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "sm__cycles_active.avg", "sm__cycles_elapsed.avg", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
            "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
            "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
            "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
            "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio"]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        res.append({k: (d.get(k), units[hdr.index(k)] if k in hdr else "") for k in keys})
    return res


def to_bytes(v, unit):
    v = float(str(v).replace(",", ""))
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--full")
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    if a.launches:
        per = launches(a.launches)
        tot = sum(sum(v) for v in per.values())
        with open(a.out + "_launches.md", "w") as f:
            f.write("# ncu launch list (gpu__time_duration.sum, --clock-control none; cold-cache, serialised)\n\n")
            f.write("| kernel | launches | total µs | mean µs | share |\n|---|---|---|---|---|\n")
            for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
                f.write(f"| `{k[:90]}` | {len(v)} | {sum(v):.1f} | {sum(v) / len(v):.2f} | {sum(v) / tot:.1%} |\n")
        print(open(a.out + "_launches.md").read())
    if a.full:
        res = full(a.full)
        step_bytes, step_us = 0.0, 0.0
        with open(a.out + "_full.md", "w") as f:
            f.write("# ncu --set full (captured launches of the bench step; serialised, cold caches)\n\n")
            for i, r in enumerate(res):
                f.write(f"## launch {i}: `{r['Kernel Name'][0][:100]}`\n\n")
                for k, (v, u) in r.items():
                    if k != "Kernel Name":
                        f.write(f"- {k}: {v} {u}\n")
                rb = to_bytes(*r["dram__bytes_read.sum"]) + to_bytes(*r["dram__bytes_write.sum"])
                step_bytes += rb
                f.write(f"- dram read+write bytes: {rb:.0f}\n\n")
                t = float(str(r["gpu__time_duration.sum"][0]).replace(",", ""))
                step_us += t / 1e3 if r["gpu__time_duration.sum"][1] == "nsecond" else t
        json.dump({"dram_bytes_per_launch": step_bytes / max(len(res), 1), "launches": len(res),
                   "source": os.path.basename(a.full), "gpu_time_us_per_launch_cold": step_us / max(len(res), 1),
                   "kernels": [r["Kernel Name"][0] for r in res],
                   "note": "dram__bytes_read.sum + dram__bytes_write.sum of the captured launch(es) of "
                           "`ncu --set full` (serialised, cold caches)"},
                  open(os.path.join(os.path.dirname(a.out), "ncu_traffic.json"), "w"), indent=1)
        print(open(a.out + "_full.md").read()[:3000])


if __name__ == "__main__":
    main()
