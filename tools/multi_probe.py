#!/usr/bin/env python3
"""Probe of the in-process multi-GPU SSSP on one GPU (a device listed several
times): path graphs (many rounds) with and without 32-bit overflow."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2401_02472_b200 as gdx  # noqa: E402
from oracle import Port  # noqa: E402

port = Port()
for n, wv in ((300, 1), (300, 1 << 27), (3000, 5)):
    u = np.arange(n - 1, dtype=np.int32)
    g = port.build_from_edges(n, u, u + 1, np.full(n - 1, wv, np.int32), False)
    exp = port.sssp(g, 0)
    for devs in ([0], [0, 0]):
        ctx = gdx.Context(devs)
        mg = gdx.MultiGraph(ctx, g)
        t0 = time.perf_counter()
        try:
            st = {}
            d = mg.sssp(0, stats=st)
            ok = np.array_equal(d, exp)
            print(f"n={n} w={wv} devs={devs}: ok={ok} {1e3 * (time.perf_counter() - t0):.1f} ms {st}",
                  flush=True)
        except Exception as e:  # noqa: BLE001
            print(f"n={n} w={wv} devs={devs}: FAILED {e} after {time.perf_counter() - t0:.1f}s",
                  flush=True)
        mg.close()
        ctx.close()
