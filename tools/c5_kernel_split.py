#!/usr/bin/env python3
"""Per-kernel split of one SSSP call (scan mode: host-driven rounds, each
kernel timed with CUDA events on the library's stream).

  python tools/c5_kernel_split.py [--scale 26]   # 18 = C1's shape (counter twin)
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2401_02472_b200 as gdx  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=26)
a = ap.parse_args()
os.environ["GDX_SSSP_MODE"] = "scan"
dg = gdx.DeviceGraph.generate("rmat", 1 << a.scale, 1 << (a.scale + 4), seed=1, directed=False,
                              weights=(1, 100))
dg.sssp(0)
dg.profile(True)
for i in range(2):
    dg.profile_reset()
    st = {}
    dg.sssp(0, stats=st)
    print(st["rounds"], dg.profile_read())
