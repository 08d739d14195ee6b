#!/usr/bin/env python3
"""How much would a lane-strided PageRank pass A gain over sorted renumbered
rows?  The random contrib gather of C2 timed with torch.index_select (thread i
gathers edge i: a warp instruction covers 32 consecutive edges) on
(a) the generator's ids, (b) ids renumbered by descending out-degree with each
row's sources sorted (built by gdx_graph_build_from_edges), against the
library's pass A on (b) (a lane owns 8 consecutive edges)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2401_02472_b200 as gdx  # noqa: E402


def timeit(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def gather_ms(g, n):
    (src,) = g.device_arrays(["rev_srcs"])
    contrib = torch.rand(n, dtype=torch.float64, device="cuda")
    out = torch.empty(src.numel(), dtype=torch.float64, device="cuda")
    return timeit(lambda: torch.index_select(contrib, 0, src, out=out))


def pass_a_ms(g):
    g.pagerank(0.85, 1e-6, 100)
    g.profile(True)
    g.profile_reset()
    _, r = g.pagerank(0.85, 1e-6, 100)
    p = g.profile_read()
    g.profile(False)
    return p["pr_edges"][0] / r


def main():
    os.environ["GDX_RELABEL"] = "0"  # the library's own renumbering off: explicit graphs here
    g = gdx.DeviceGraph.generate("rmat", 1 << 24, 1 << 28, seed=1, directed=True)
    n = g.n
    print(f"(a) generator ids: index_select {gather_ms(g, n):.3f} ms, pass A {pass_a_ms(g):.3f} ms",
          flush=True)
    h = g.download(("offsets", "rev_offsets", "rev_srcs"))
    g.close()
    order = np.argsort(-np.diff(h.offsets), kind="stable")
    newid = np.empty(n, np.int32)
    newid[order] = np.arange(n, dtype=np.int32)
    dst = np.repeat(np.arange(n, dtype=np.int32), np.diff(h.rev_offsets))
    g2 = gdx.DeviceGraph.build_from_edges(n, newid[h.rev_srcs], newid[dst], None, directed=True)
    print(f"(b) renumbered, sorted rows: index_select {gather_ms(g2, n):.3f} ms, "
          f"pass A {pass_a_ms(g2):.3f} ms", flush=True)


if __name__ == "__main__":
    main()
