#!/usr/bin/env python3
"""A/B of the SSSP executions (GDX_SSSP_MODE=graph|persistent|scan) on a
low-diameter RMAT graph and a high-diameter road-like grid."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2401_02472_b200 as gdx  # noqa: E402

graphs = {
    "rmat20": gdx.DeviceGraph.generate("rmat", 1 << 20, 16 << 20, seed=1, directed=False,
                                       weights=(1, 100)),
    "grid2000": gdx.DeviceGraph.generate("grid", 2000, seed=1, keep=0.55, directed=False,
                                         weights=(1, 100)),
}
for name, g in graphs.items():
    src = 0 if name.startswith("rmat") else 1000 * 2000 + 1000  # grid centre
    for mode in ("graph", "persistent", "scan"):
        os.environ["GDX_SSSP_MODE"] = mode
        g.sssp(src)
        st = {}
        g.profile(True)
        g.profile_reset()
        t0 = time.perf_counter()
        g.sssp(src, stats=st)
        wall = (time.perf_counter() - t0) * 1e3
        dev = sum(v[0] for v in g.profile_read().values())
        g.profile(False)
        print(f"{name} {mode}: {wall:.1f} ms wall, {dev:.2f} ms device, rounds={st['rounds']}",
              flush=True)
