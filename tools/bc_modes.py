#!/usr/bin/env python3
"""A/B of the BC executions (GDX_BC_MODE=grid|cta) on RMAT and grid graphs for
small source counts."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2401_02472_b200 as gdx  # noqa: E402


def main():
    graphs = {
        "rmat20": gdx.DeviceGraph.generate("rmat", 1 << 20, 16 << 20, seed=1, directed=False),
        "grid2000": gdx.DeviceGraph.generate("grid", 2000, seed=1, keep=0.55, directed=False),
    }
    for name, g in graphs.items():
        deg = np.diff(g.download().offsets)
        cand = np.flatnonzero(deg > 0)
        for ns in (1, 4, 16, 64):
            src = sorted(np.random.default_rng(ns).choice(cand, ns, replace=False).tolist())
            for mode in ("grid", "cta"):
                os.environ["GDX_BC_MODE"] = mode
                g.bc(src)
                t0 = time.perf_counter()
                st = {}
                g.bc(src, stats=st)
                dt = time.perf_counter() - t0
                print(f"{name} sources={ns} mode={mode}: {dt * 1e3:.1f} ms levels={st['rounds']}",
                      flush=True)


if __name__ == "__main__":
    main()
