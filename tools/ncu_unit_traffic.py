#!/usr/bin/env python3
"""DRAM bytes per unit of work (one SSSP / TC / BC call, one PR round) from an
ncu metrics log of every kernel of that unit, for bench.py's roofline.traffic.

  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none -k regex:k_sssp --csv --log-file gpurun_out/traffic_sssp_c5.csv \
      env GDX_SSSP_MODE=scan python tools/kernel_driver.py --algo sssp26 --reps 2
  python tools/ncu_unit_traffic.py --key sssp_c5_call --log gpurun_out/traffic_sssp_c5.csv \
      --start k_sssp_scan_init --units 2

Kernels are grouped into units by `--start` (the first kernel of a unit; PR:
k_pr_edges of each round); the LAST complete unit is reported (the earlier
ones are warm-up).  Kernels inside CUDA graphs with conditional nodes cannot
be replayed one by one, so SSSP is captured in the host-driven loop
(GDX_SSSP_MODE=scan): the same kernels the graph runs.
"""
import argparse
import csv
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
        "ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3, "s": 1.0}


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hi]
    ii, ki, mi, vi, ui = (hdr.index("ID"), hdr.index("Kernel Name"), hdr.index("Metric Name"),
                          hdr.index("Metric Value"), hdr.index("Metric Unit"))
    out = {}
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        d = out.setdefault(int(r[ii]), {"kernel": r[ki].split("(")[0]})
        d[r[mi]] = float(r[vi].replace(",", "")) * UNIT.get(r[ui], 1.0)
    return [out[k] for k in sorted(out)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--key", required=True)
    ap.add_argument("--log", required=True)
    ap.add_argument("--start", required=True, help="substring of the first kernel of a unit")
    ap.add_argument("--unit", default="call")
    a = ap.parse_args()
    ls = launches(a.log)
    units, cur = [], None
    for d in ls:
        if a.start in d["kernel"]:
            cur = []
            units.append(cur)
        if cur is not None:
            cur.append(d)
    if a.unit == "round":
        # PR: rounds enqueued after the vote settled exit at once -- report the
        # median of the rounds that did work (>= half the longest round)
        dur = [sum(d.get("gpu__time_duration.sum", 0.0) for d in x) for x in units]
        work = sorted((x for x, t in zip(units, dur) if t >= 0.5 * max(dur)),
                      key=lambda x: sum(d.get("dram__bytes_read.sum", 0.0) for d in x))
        u = work[len(work) // 2]
    else:
        u = units[-1]
    rd = sum(d.get("dram__bytes_read.sum", 0.0) for d in u)
    wr = sum(d.get("dram__bytes_write.sum", 0.0) for d in u)
    t = sum(d.get("gpu__time_duration.sum", 0.0) for d in u)
    kern = {}
    for d in u:
        k = kern.setdefault(d["kernel"], {"launches": 0, "dram_bytes": 0.0, "ms": 0.0})
        k["launches"] += 1
        k["dram_bytes"] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
        k["ms"] += d.get("gpu__time_duration.sum", 0.0) * 1e3
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    summ = json.load(open(p)) if os.path.exists(p) else {}
    summ[a.key] = {"unit": a.unit, "dram_bytes_per_unit": rd + wr, "dram_read": rd,
                   "dram_write": wr, "ncu_ms_per_unit": t * 1e3, "kernels": kern,
                   "source": os.path.basename(a.log),
                   "how": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,"
                          "dram__bytes_write.sum --clock-control none (cold, serialised replays)"}
    json.dump(summ, open(p, "w"), indent=1)
    print(a.key, json.dumps(summ[a.key]))


if __name__ == "__main__":
    main()
