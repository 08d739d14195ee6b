#!/usr/bin/env python3
"""Summarise ncu captures into profiles/ (tracked).

  python tools/make_profiles.py --round r01 \
      --rep pr=gpurun_out/ncu_pr.ncu-rep --rep sssp=... \
      --launches gpurun_out/launches_pr.csv

Writes profiles/ncu_summary.json (per kernel: duration, DRAM bytes per launch,
hit rates -- bench.py reads `dram_bytes_per_launch` for roofline.traffic) and
profiles/ncu_summary_<round>.md (human-readable, with the hottest source lines).
"""
import argparse
import csv
import io
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, HERE)

from ncu_hot import hot_lines  # noqa: E402

METRICS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_peak",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "l1tex__t_sector_hit_rate.pct": "l1_hit_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_throughput_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
        "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {"kernel": vals[hdr.index("Kernel Name")]}
    for m, k in METRICS.items():
        if m not in hdr:
            continue
        i = hdr.index(m)
        v = float(vals[i].replace(",", ""))
        u = units[i]
        if u in UNIT:
            v *= UNIT[u]
            if k == "duration":
                k = "duration_s"
        d[k] = v
    d["dram_bytes_per_launch"] = d.get("dram_read", 0.0) + d.get("dram_write", 0.0)
    return d


def launches(path):
    """Per-kernel launch count and total time from an ncu --metrics
    gpu__time_duration.sum CSV log."""
    rows = list(csv.reader(open(path)))
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hdr_i]
    ki, mi, vi, ui = (hdr.index("Kernel Name"), hdr.index("Metric Name"),
                      hdr.index("Metric Value"), hdr.index("Metric Unit"))
    agg = {}
    for r in rows[hdr_i + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0]
        t = float(r[vi].replace(",", "")) * UNIT.get(r[ui], 1e-9)
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += t
    total = sum(v[1] for v in agg.values()) or 1.0
    return {k: {"launches": v[0], "total_ms": v[1] * 1e3, "share": v[1] / total}
            for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", default="r01")
    ap.add_argument("--rep", action="append", default=[], help="name=path.ncu-rep")
    ap.add_argument("--launches", default=None)
    a = ap.parse_args()
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    summary_path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    summary = json.load(open(summary_path)) if os.path.exists(summary_path) else {}
    md = [f"# ncu summaries ({a.round})", "",
          "Captured with `ncu --set full --clock-control none --import-source on` on one B200",
          "(`tools/kernel_driver.py`, BASELINE configs). Durations are ncu replays (cold-cache,",
          "serialised); bench.py's live CUDA-event timings are the reported numbers.", ""]
    for spec in a.rep:
        name, path = spec.split("=", 1)
        d = raw(path)
        key = name  # the kernel name bench.py's roofline looks up
        summary[key] = {k: v for k, v in d.items()}
        summary[key]["source"] = os.path.basename(path)
        md.append(f"## {name}: `{d['kernel'][:90]}`")
        md.append("")
        md.append("| metric | value |")
        md.append("|---|---|")
        for k, v in d.items():
            if k == "kernel":
                continue
            md.append(f"| {k} | {v:.4g} |" if isinstance(v, float) else f"| {k} | {v} |")
        md.append("")
        md.append("Hottest source lines (share of warp-stall samples):")
        md.append("")
        md.append("```")
        md.extend(hot_lines(path, 12))
        md.append("```")
        md.append("")
    if a.launches:
        L = launches(a.launches)
        summary["launch_list"] = L
        md.append("## Launch list (`ncu --metrics gpu__time_duration.sum`)")
        md.append("")
        md.append("| kernel | launches | total ms | share |")
        md.append("|---|---|---|---|")
        for k, v in L.items():
            md.append(f"| {k} | {v['launches']} | {v['total_ms']:.3f} | {v['share']:.3f} |")
        md.append("")
    json.dump(summary, open(summary_path, "w"), indent=1)
    with open(os.path.join(ROOT, "profiles", f"ncu_summary_{a.round}.md"), "w") as f:
        f.write("\n".join(md) + "\n")
    print("wrote", summary_path)


if __name__ == "__main__":
    main()
