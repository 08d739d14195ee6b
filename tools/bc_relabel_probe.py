#!/usr/bin/env python3
"""C4 BC (64 sources, 4899^2 grid keep 0.55) against the same graph with its
vertices renumbered for locality: (a) BFS order from vertex 0 (Cuthill-McKee
style: vertices of one BFS level contiguous), (b) 2-D tiles of the grid
(8 x 8 blocks of the row-major ids), to size what a locality renumbering would
buy a latency-bound level loop.  Same kernels; scores compared through the
permutation."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2401_02472_b200 as gdx  # noqa: E402


def run(dg, sources, label):
    out = torch.empty(dg.n, dtype=torch.float64, device="cuda")
    dg.bc(sources, out=out)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dg.bc(sources, out=out)
    torch.cuda.synchronize()
    print(f"{label}: {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)
    return out.cpu().numpy()


def relabelled(h, newid):
    n = h.n
    deg = np.diff(h.offsets)
    u = np.repeat(np.arange(n, dtype=np.int32), deg)
    return gdx.DeviceGraph.build_from_edges(n, newid[u], newid[h.dests], None, directed=True)


def main():
    side = 4899
    dg = gdx.DeviceGraph.generate("grid", side, seed=1, keep=0.55, directed=False)
    h = dg.download(("offsets", "dests"))
    n = h.n
    deg = np.diff(h.offsets)
    rng = np.random.default_rng(1)
    cand = np.flatnonzero(deg > 0)
    sources = sorted(rng.choice(cand, size=64, replace=False).tolist())
    b0 = run(dg, sources, "row-major (as generated)")
    # (a) BFS order from the first source: unweighted SSSP distances, stable sort
    d = dg.sssp(sources[0])
    dg.close()
    order = np.lexsort((np.arange(n), d))
    newid = np.empty(n, np.int32)
    newid[order] = np.arange(n, dtype=np.int32)
    g = relabelled(h, newid)
    b = run(g, [int(newid[s]) for s in sources], "BFS order")
    print("  max rel diff", float(np.max(np.abs(b[newid] - b0) / np.maximum(np.abs(b0), 1e-12))))
    g.close()
    # (b) 8 x 8 tiles of the grid (ids are r * side + c)
    r, c = np.divmod(np.arange(n, dtype=np.int64), side)
    key = ((r // 8) * ((side + 7) // 8) + c // 8) * 64 + (r % 8) * 8 + c % 8
    order = np.argsort(key, kind="stable")
    newid[order] = np.arange(n, dtype=np.int32)
    g = relabelled(h, newid)
    b = run(g, [int(newid[s]) for s in sources], "8x8 tiles")
    print("  max rel diff", float(np.max(np.abs(b[newid] - b0) / np.maximum(np.abs(b0), 1e-12))))


if __name__ == "__main__":
    main()
