#!/usr/bin/env python3
"""Time the PageRank round kernels on the C2 graph under environment A/B
knobs (e.g. GDX_PR_GRID_CAP=16,64).

  python tools/pr_variants.py [--env GDX_PR_GRID_CAP=16,32,64] [--scale 24]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import paper_2401_02472_b200 as gdx  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--env", default="", help="NAME=v1,v2,... (one run per value)")
    ap.add_argument("--scale", type=int, default=24)
    ap.add_argument("--reps", type=int, default=4)
    a = ap.parse_args()
    name, vals = (a.env.split("=", 1) + [""])[:2] if a.env else ("", "default")
    ref = None
    for v in vals.split(","):
        if name:
            os.environ[name] = v
        g = gdx.DeviceGraph.generate("rmat", 1 << a.scale, 16 << a.scale, seed=1, directed=True)
        g.profile(True)
        g.pagerank(0.85, 1e-6, 100)
        g.profile_reset()
        t0 = time.perf_counter()
        for _ in range(a.reps):
            r, rounds = g.pagerank(0.85, 1e-6, 100)
        wall = (time.perf_counter() - t0) / a.reps
        prof = g.profile_read()
        ms = sum(x[0] for k, x in prof.items() if k != "pr_init")
        per_round = ms / (rounds * a.reps)
        parts = " ".join(f"{k}={x[0] / (rounds * a.reps):.3f}" for k, x in prof.items()
                         if k != "pr_init")
        gbs = (12.0 * g.m + 32.0 * g.n) / (per_round * 1e-3) / 1e9
        diff = 0.0 if ref is None else float(np.max(np.abs(r - ref) / np.abs(ref)))
        ref = r if ref is None else ref
        print(f"{name or 'default'}={v}: rounds={rounds} round kernels {per_round:.3f} ms/round "
              f"[{parts}] ({gbs:.0f} GB/s algorithmic) wall {wall * 1e3:.1f} ms/run  "
              f"maxrel vs first {diff:.2e}", flush=True)
        g.close()


if __name__ == "__main__":
    main()
