#!/usr/bin/env python3
"""Time the pieces of bench.py's e2e PageRank step (graph create from pinned
host CSR, first call incl. plan build, steady-state call, close)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2401_02472_b200 as gdx  # noqa: E402


def main():
    dg = gdx.DeviceGraph.generate("rmat", 1 << 24, 1 << 28, seed=1, directed=True)
    h = dg.download()
    n, m = dg.n, dg.m
    dg.close()
    pin = {k: torch.from_numpy(getattr(h, k)).pin_memory() for k in ("offsets", "rev_offsets", "rev_srcs")}
    out = torch.empty(n, dtype=torch.float64).pin_memory()

    class V:
        pass

    v = V()
    v.n, v.m, v.directed = n, m, True
    v.offsets, v.rev_offsets, v.rev_srcs = pin["offsets"], pin["rev_offsets"], pin["rev_srcs"]
    v.dests = v.weights = v.rev_eid = None
    for it in range(3):
        t0 = time.perf_counter()
        g = gdx.DeviceGraph.from_csr(v)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        g.profile(True)
        g.pagerank(0.85, 1e-6, 100, out=out)
        t2 = time.perf_counter()
        g.pagerank(0.85, 1e-6, 100, out=out)
        t3 = time.perf_counter()
        prof = g.profile_read()
        g.close()
        t4 = time.perf_counter()
        print(f"create {1e3 * (t1 - t0):.1f} ms, first PR {1e3 * (t2 - t1):.1f} ms, "
              f"second PR {1e3 * (t3 - t2):.1f} ms, close {1e3 * (t4 - t3):.1f} ms; "
              + " ".join(f"{k}={v[0]:.2f}ms/{v[1]}" for k, v in prof.items()), flush=True)


if __name__ == "__main__":
    main()
