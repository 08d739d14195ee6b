#!/usr/bin/env python3
"""A/B the PageRank round kernels (GDX_PR_VARIANT) on the C2 graph.

  python tools/pr_variants.py [--variants 1,3,4] [--scale 24]
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
    ap.add_argument("--variants", default="1,3,4")
    ap.add_argument("--scale", type=int, default=24)
    ap.add_argument("--reps", type=int, default=4)
    a = ap.parse_args()
    ref = None
    for v in a.variants.split(","):
        os.environ["GDX_PR_VARIANT"] = v
        g = gdx.DeviceGraph.generate("rmat", 1 << a.scale, 16 << a.scale, seed=1, directed=True)
        g.profile(True)
        g.pagerank(0.85, 1e-6, 100)
        g.profile_reset()
        t0 = time.perf_counter()
        for _ in range(a.reps):
            r, rounds = g.pagerank(0.85, 1e-6, 100)
        wall = (time.perf_counter() - t0) / a.reps
        prof = g.profile_read()
        ms = sum(v[0] for k, v in prof.items() if k != "pr_init")
        per_round = ms / (rounds * a.reps)
        parts = " ".join(f"{k}={v[0] / (rounds * a.reps):.3f}" for k, v in prof.items() if k != "pr_init")
        gbs = (12.0 * g.m + 32.0 * g.n) / (per_round * 1e-3) / 1e9
        diff = 0.0 if ref is None else float(np.max(np.abs(r - ref) / np.abs(ref)))
        ref = r if ref is None else ref
        print(f"variant {v}: rounds={rounds} round kernels {per_round:.3f} ms/round [{parts}] "
              f"({gbs:.0f} GB/s algorithmic) wall {wall * 1e3:.1f} ms/run  maxrel vs first {diff:.2e}",
              flush=True)
        g.close()


if __name__ == "__main__":
    main()
