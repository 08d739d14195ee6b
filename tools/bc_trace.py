#!/usr/bin/env python3
"""Per-level latency breakdown of the CTA-cluster BC kernel on C4 (GDX_BC_TRACE):
slot 0's time per level step against the level's item count, forward and
backward, for each cluster size in --clusters.

  python tools/bc_trace.py [--sources 64] [--clusters 1,2]
"""
import argparse
import os
import sys
import tempfile
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2401_02472_b200 as gdx  # noqa: E402


def summarise(path):
    t = np.loadtxt(path, dtype=np.float64, ndmin=2)
    rest = t[t[:, 1] == 1 << 30]
    t = t[t[:, 1] != 1 << 30]
    fwd, bwd = t[t[:, 1] >= 0], t[t[:, 1] < 0] * [1, -1]
    out = {"restore_us": (rest[:, 0] / 1e3).round(1).tolist()}
    for name, x in (("fwd", fwd), ("bwd", bwd)):  # noqa: B007
        if len(x) == 0:
            continue
        ns, items = x[:, 0], x[:, 1]
        slope, icpt = np.polyfit(items, ns, 1)
        qs = np.quantile(items, [0.1, 0.5, 0.9])
        out[name] = dict(steps=len(x), mean_us=ns.mean() / 1e3, total_ms=ns.sum() / 1e6,
                         intercept_us=icpt / 1e3, ns_per_item=slope,
                         items_p10_50_90=[int(q) for q in qs])
        for lo, hi in ((0, 512), (512, 2048), (2048, 4096), (4096, 1 << 30)):
            m = (items >= lo) & (items < hi)
            if m.any():
                out[name][f"items[{lo},{hi})"] = f"{m.sum()} steps, {ns[m].mean() / 1e3:.2f} us"
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sources", type=int, default=64)
    ap.add_argument("--clusters", default="1,2")
    ap.add_argument("--side", type=int, default=4899)
    a = ap.parse_args()
    g = gdx.DeviceGraph.generate("grid", a.side, seed=1, keep=0.55, directed=False)
    deg = np.diff(g.download().offsets)
    src = sorted(np.random.default_rng(1).choice(np.flatnonzero(deg > 0), a.sources,
                                                 replace=False).tolist())
    os.environ["GDX_BC_MODE"] = "cta"
    for cs in a.clusters.split(","):
        os.environ["GDX_BC_CLUSTER"] = cs
        os.environ.pop("GDX_BC_TRACE", None)
        g.bc(src)
        t0 = time.perf_counter()
        st = {}
        g.bc(src, stats=st)
        dt = time.perf_counter() - t0
        path = os.path.join(tempfile.gettempdir(), f"bc_trace_{cs}.txt")
        os.environ["GDX_BC_TRACE"] = path
        g.bc(src)
        print(f"cluster={cs}: {a.sources} sources {dt * 1e3:.1f} ms, max levels {st['rounds']}",
              flush=True)
        for k, v in summarise(path).items():
            print(f"  {k}: {v}", flush=True)
        os.environ.pop("GDX_BC_TRACE", None)


if __name__ == "__main__":
    main()
