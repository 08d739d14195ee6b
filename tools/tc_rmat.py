#!/usr/bin/env python3
"""TC on skewed graphs (RMAT, undirected): time and count, to watch the
oriented kernel's hub handling (C3 is uniform)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2401_02472_b200 as gdx  # noqa: E402

for directed in (False, True):
    for sc in (18, 20, 22):
        g = gdx.DeviceGraph.generate("rmat", 1 << sc, 16 << sc, seed=1, directed=directed)
        g.tc()
        t0 = time.perf_counter()
        c = g.tc()
        print(f"rmat-{sc} {'directed' if directed else 'undirected'} m={g.m}: {c} triangles in "
              f"{(time.perf_counter() - t0) * 1e3:.1f} ms", flush=True)
        g.close()
