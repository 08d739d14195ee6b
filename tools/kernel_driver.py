#!/usr/bin/env python3
"""Minimal driver for ncu captures: builds one BASELINE config graph on the GPU
and calls one entry point `--reps` times (no timing, no oracle).

  ncu --set full --clock-control none --import-source on -k regex:pr_tiles -s 2 -c 1 \
      -o gpurun_out/pr python tools/kernel_driver.py --algo pr
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
    ap.add_argument("--algo", default="pr", choices=["pr", "sssp", "sssp26", "tc", "bc"])
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--bc-sources", type=int, default=64)
    a = ap.parse_args()
    _orig_generate = gdx.DeviceGraph.generate

    def generate(*args, **kw):  # enable per-kernel event timing on every graph
        g = _orig_generate(*args, **kw)
        g.profile(True)
        graphs.append(g)
        return g

    graphs = []
    gdx.DeviceGraph.generate = generate
    if a.algo == "pr":
        g = gdx.DeviceGraph.generate("rmat", 1 << 24, 1 << 28, seed=1, directed=True)
        for _ in range(a.reps):
            print(g.pagerank(0.85, 1e-6, 100)[1])
        graphs_pr = graphs  # noqa: F841
    elif a.algo in ("sssp", "sssp26"):
        if a.algo == "sssp":  # C1: the reference's own graph, as bench.py
            u, v = gdx.gen_rmat_edges(1 << 18, 1 << 22, 1)
            g = gdx.DeviceGraph.build_from_edges(1 << 18, u, v, None, directed=False)
            g.profile(True)
            graphs.append(g)
            g.set_random_weights(1, 100, 1)
        else:
            g = gdx.DeviceGraph.generate("rmat", 1 << 26, 1 << 30, seed=1, directed=False,
                                         weights=(1, 100))
        for _ in range(a.reps):
            st = {}
            t0 = time.perf_counter()
            g.sssp(0, stats=st)
            print(f"{(time.perf_counter() - t0) * 1e3:.3f} ms", st, flush=True)
    elif a.algo == "tc":
        g = gdx.DeviceGraph.generate("uniform", 1 << 24, 1 << 27, seed=1, directed=False)
        for _ in range(a.reps):
            print(g.tc())
    else:
        g = gdx.DeviceGraph.generate("grid", 4899, seed=1, keep=0.55, directed=False)
        h = g.download()
        cand = np.flatnonzero(np.diff(h.offsets) > 0)
        src = sorted(np.random.default_rng(1).choice(cand, a.bc_sources, replace=False).tolist())
        for _ in range(a.reps):
            st = {}
            t0 = time.perf_counter()
            g.bc(src, stats=st)
            print(f"{(time.perf_counter() - t0) * 1e3:.1f} ms", st, flush=True)


    for g in graphs:
        for k, (ms, n) in sorted(g.profile_read().items()):
            print(f"kernel {k}: {ms / max(n, 1):.4f} ms avg over {n} launches")


if __name__ == "__main__":
    main()
