#!/usr/bin/env python3
"""PageRank pass A on the C2 graph against the same graph with every vertex
renumbered by descending out-degree (the gathered contrib array then holds the
hubs -- the sources most in-edges read -- in the fewest lines), to size what a
relabelling plan cached on the handle would buy.  Same kernels, same rounds."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2401_02472_b200 as gdx  # noqa: E402


def run(dg, label, reps=5):
    dg.pagerank(0.85, 1e-6, 100)
    dg.profile(True)
    dg.profile_reset()
    rounds = 0
    torch.cuda.synchronize()
    for _ in range(reps):
        _, r = dg.pagerank(0.85, 1e-6, 100)
        rounds += r
    prof = dg.profile_read()
    dg.profile(False)
    ms = {k: v[0] / rounds for k, v in prof.items()}
    print(label, "rounds", rounds // reps, " ".join(f"{k} {v:.4f}" for k, v in sorted(ms.items())),
          "ms/round", flush=True)


def main():
    g = gdx.DeviceGraph.generate("rmat", 1 << 24, 1 << 28, seed=1, directed=True)
    run(g, "original")
    h = g.download(("offsets", "rev_offsets", "rev_srcs"))
    n = h.n
    g.close()
    dst = np.repeat(np.arange(n, dtype=np.int32), np.diff(h.rev_offsets))
    src = h.rev_srcs
    for key in ("out", "in"):
        deg = np.diff(h.offsets) if key == "out" else np.diff(h.rev_offsets)
        order = np.argsort(-deg, kind="stable")  # new id -> old id
        newid = np.empty(n, np.int32)
        newid[order] = np.arange(n, dtype=np.int32)
        g2 = gdx.DeviceGraph.build_from_edges(n, newid[src], newid[dst], None, directed=True)
        run(g2, f"relabel-by-{key}-degree")
        g2.close()
    # sources only: rows keep their order, the gathered ids are renamed
    deg = np.diff(h.offsets)
    order = np.argsort(-deg, kind="stable")
    newid = np.empty(n, np.int32)
    newid[order] = np.arange(n, dtype=np.int32)
    g3 = gdx.DeviceGraph.build_from_edges(n, newid[src], dst, None, directed=True)
    run(g3, "sources-only (rows kept; not a valid PageRank, timing only)")


if __name__ == "__main__":
    main()
