#!/usr/bin/env python3
"""Summarise an ncu report: per-CUDA-source-line warp-stall samples (from the
`cuda,sass` source view) and the headline raw metrics.

  python tools/ncu_hot.py gpurun_out/ncu_pr.ncu-rep [--top 25]
"""
import argparse
import csv
import io
import subprocess

RAW = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
       "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
       "l1tex__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
       "sm__throughput.avg.pct_of_peak_sustained_elapsed",
       "lts__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
       "launch__grid_size", "launch__block_size", "launch__occupancy_limit_registers",
       "launch__occupancy_limit_shared_mem", "smsp__inst_executed.sum"]


def run(args):
    return subprocess.run(["ncu", "-i", *args], capture_output=True, text=True).stdout


def raw_metrics(rep):
    rows = list(csv.reader(io.StringIO(run([rep, "--page", "raw", "--csv"]))))
    hdr, units = rows[0], rows[1]
    out = []
    for vals in rows[2:]:
        d = {"kernel": vals[hdr.index("Kernel Name")]}
        for m in RAW:
            if m in hdr:
                i = hdr.index(m)
                d[m] = f"{vals[i]} {units[i]}".strip()
        out.append(d)
    return out


def hot_lines(rep, top):
    text = run([rep, "--page", "source", "--csv", "--print-source", "cuda,sass"])
    rows = list(csv.reader(io.StringIO(text)))
    agg, hdr = {}, None
    for r in rows:
        if len(r) > 4 and r[0] == "Line No":
            hdr = r
            si = hdr.index("Warp Stall Sampling (All Samples)")
            stall_cols = [(i, h) for i, h in enumerate(hdr)
                          if h.startswith("stall_") and "Not Issued" not in h]
            continue
        if hdr is None or not r or not r[0].isdigit():
            continue  # SASS rows carry no line number; CUDA rows hold the line totals
        try:
            s = int(r[si] or 0)
        except ValueError:
            continue
        key = f"{r[0]}: {r[1].strip()[:90]}"
        a = agg.setdefault(key, {"samples": 0})
        a["samples"] += s
        for i, h in stall_cols:
            try:
                v = int(r[i] or 0)
            except ValueError:
                v = 0
            if v:
                a[h] = a.get(h, 0) + v
    total = sum(a["samples"] for a in agg.values()) or 1
    lines = sorted(agg.items(), key=lambda kv: -kv[1]["samples"])[:top]
    out = []
    for k, a in lines:
        top3 = sorted(((v, h) for h, v in a.items() if h != "samples"), reverse=True)[:3]
        out.append(f"{100.0 * a['samples'] / total:5.1f}%  {k}   " +
                   ", ".join(f"{h[6:]}={v}" for v, h in top3))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--top", type=int, default=25)
    a = ap.parse_args()
    for d in raw_metrics(a.rep):
        print(d["kernel"][:100])
        for k, v in d.items():
            if k != "kernel":
                print(f"  {k:62s} {v}")
    print("hot source lines (share of warp-stall samples):")
    for line in hot_lines(a.rep, a.top):
        print("  " + line)


if __name__ == "__main__":
    main()
