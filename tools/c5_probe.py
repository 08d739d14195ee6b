#!/usr/bin/env python3
"""C5 (BASELINE config 5): SSSP on RMAT scale-26 (2^30 draws, undirected,
weights U[1,100]) on one B200: build time, SSSP time, and a size-independent
correctness certificate (every edge satisfies d[v] <= d[u] + w, every reached
vertex has a tight in-edge, d[src] = 0)."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2401_02472_b200 as gdx  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=26)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    t0 = time.perf_counter()
    g = gdx.DeviceGraph.generate("rmat", 1 << a.scale, 16 << a.scale, seed=1, directed=False,
                                 weights=(1, 100))
    torch.cuda.synchronize()
    print(f"build: n={g.n} m={g.m} in {time.perf_counter() - t0:.1f}s "
          f"(free {torch.cuda.mem_get_info()[0] / 2**30:.1f} GiB)", flush=True)
    out = torch.empty(g.n, dtype=torch.int64, device="cuda")
    g.profile(True)
    for r in range(a.reps):
        st = {}
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        g.sssp(0, out=out, stats=st)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t1
        print(f"sssp: {dt * 1e3:.1f} ms wall, rounds {st['rounds']}, E_vis/m "
              f"{st['edges_visited'] / g.m:.2f}, GTEPS {g.m / dt / 1e9:.1f}", flush=True)
    print(g.profile_read())
    # certificate
    off, dst, w = g.device_arrays(["offsets", "dests", "weights"])
    INF = (2**63 - 1) // 2
    d = out
    n = g.n
    tight = torch.zeros(n, dtype=torch.bool, device="cuda")
    ok = True
    chunk = 1 << 27
    deg = (off[1:] - off[:-1]).long()
    for e0 in range(0, g.m, chunk):
        e1 = min(g.m, e0 + chunk)
        eid = torch.arange(e0, e1, device="cuda", dtype=torch.int64)
        src = torch.searchsorted(off.long(), eid, right=True) - 1
        du = d[src]
        dv = d[dst[e0:e1].long()]
        fin = du < INF
        cand = du + w[e0:e1].long()
        ok &= bool(torch.all(~fin | (dv <= cand)))
        tight.index_fill_(0, dst[e0:e1].long()[fin & (dv == cand)], True)
    reached = d < INF
    ok &= int(d[0]) == 0
    tight[0] = True
    ok &= bool(torch.all(~reached | tight))
    print(f"certificate: {'OK' if ok else 'FAILED'}; reached {int(reached.sum())} of {n}, "
          f"max dist {int(d[reached].max())}")


if __name__ == "__main__":
    main()
