#!/usr/bin/env python3
"""Measure the random-gather floor of a PageRank round on the C2 graph with
plain torch ops (index_select over rev_srcs), with and without relabelling
vertices by out-degree, to size the headroom of the PR kernel."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2401_02472_b200 as gdx  # noqa: E402


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    g = gdx.DeviceGraph.generate("rmat", 1 << 24, 1 << 28, seed=1, directed=True)
    h = g.download()
    n, m = h.n, h.m
    src = torch.from_numpy(h.rev_srcs.astype(np.int64)).cuda()
    src32 = torch.from_numpy(h.rev_srcs).cuda()
    contrib = torch.rand(n, dtype=torch.float64, device="cuda")
    out = torch.empty(m, dtype=torch.float64, device="cuda")
    t = timeit(lambda: torch.index_select(contrib, 0, src32, out=out))
    print(f"index_select gather m={m}: {t:.3f} ms  ({(12 * m) / t / 1e6:.0f} GB/s of 4B idx + 8B val + 8B out)")
    t = timeit(lambda: contrib[src].sum())
    print(f"gather+sum: {t:.3f} ms")
    outdeg = np.diff(h.offsets)
    order = np.argsort(-outdeg, kind="stable")  # new id -> old id
    newid = np.empty(n, np.int64)
    newid[order] = np.arange(n)
    src2 = torch.from_numpy(newid[h.rev_srcs].astype(np.int32)).cuda()
    t = timeit(lambda: torch.index_select(contrib, 0, src2, out=out))
    print(f"index_select gather, sources relabelled by out-degree: {t:.3f} ms")
    c32 = contrib.float()
    o32 = torch.empty(m, dtype=torch.float32, device="cuda")
    t = timeit(lambda: torch.index_select(c32, 0, src32, out=o32))
    print(f"index_select gather of an f32 array (L2-resident 4n bytes): {t:.3f} ms")
    t = timeit(lambda: torch.index_select(c32, 0, src2, out=o32))
    print(f"index_select gather f32, relabelled: {t:.3f} ms")
    # sources compacted to the vertices with out-edges (order kept): the gathered
    # array shrinks to the non-dangling vertices
    nd = outdeg > 0
    cidx = np.cumsum(nd) - 1
    srcc = torch.from_numpy(cidx[h.rev_srcs].astype(np.int32)).cuda()
    cc = torch.rand(int(nd.sum()), dtype=torch.float64, device="cuda")
    t = timeit(lambda: torch.index_select(cc, 0, srcc, out=out))
    print(f"index_select gather, sources compacted to {int(nd.sum())} non-dangling ({cc.numel() * 8 / 2**20:.0f} MB): {t:.3f} ms")
    indeg = np.diff(h.rev_offsets)
    print(f"in-degree: zero={np.mean(indeg == 0):.3f} max={indeg.max()} ; out-degree zero={np.mean(outdeg == 0):.3f} max={outdeg.max()}")
    hot = np.bincount(h.rev_srcs, minlength=n)
    srt = np.sort(hot)[::-1]
    for k in (1 << 13, 1 << 14, 1 << 15, 1 << 16, 1 << 20, 1 << 22):
        print(f"top {k} sources cover {srt[:k].sum() / m:.3f} of gathers ({k * 8 / 2**20:.0f} MB of contrib)")


if __name__ == "__main__":
    main()
