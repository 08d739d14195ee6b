#!/usr/bin/env python3
"""SSSP on an RMAT graph against the same graph with every vertex renumbered
by descending degree (hub distances packed into the fewest lines of the
gathered dist array), to size what a relabelling plan cached on the handle
would buy.  Same kernels; distances compared through the permutation."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2401_02472_b200 as gdx  # noqa: E402


def run(dg, src, label, reps=5):
    out = torch.empty(dg.n, dtype=torch.int64, device="cuda")
    dg.sssp(src, out=out)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        st = {}
        dg.sssp(src, out=out, stats=st)
    b.record()
    torch.cuda.synchronize()
    print(label, f"{a.elapsed_time(b) / reps:.3f} ms/call rounds {st['rounds']} "
          f"edges/m {st['edges_visited'] / dg.m:.3f}", flush=True)
    return out.cpu().numpy()


def main():
    scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
    n = 1 << scale
    g = gdx.DeviceGraph.generate("rmat", n, 16 * n, seed=1, directed=False, weights=(1, 100))
    d0 = run(g, 0, f"rmat-{scale} original")
    h = g.download(("offsets", "dests", "weights"))
    g.close()
    deg = np.diff(h.offsets)
    order = np.argsort(-deg, kind="stable")  # new id -> old id
    newid = np.empty(n, np.int32)
    newid[order] = np.arange(n, dtype=np.int32)
    u = np.repeat(np.arange(n, dtype=np.int32), deg)
    g2 = gdx.DeviceGraph.build_from_edges(n, newid[u], newid[h.dests], h.weights, directed=True)
    del u
    d1 = run(g2, int(newid[0]), f"rmat-{scale} relabelled by degree")
    print("distances equal through the permutation:", bool(np.array_equal(d1[newid], d0)))


if __name__ == "__main__":
    main()
