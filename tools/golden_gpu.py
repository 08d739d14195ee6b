#!/usr/bin/env python3
"""The reference's own GPU realisation (its generated CUDA units,
proj/tests/golden/*/cuda/*.cu, compiled unchanged into oracle/_ref/libgolden.so
by `make -C oracle golden`) timed beside this backend on the same B200 and the
same BASELINE graphs, with the results cross-checked.

Each golden call uploads the graph, runs with a host round trip per
iteration/level and downloads the result (e.g. pr_cuda.cu:150-224), so its wall
time is compared with ours end to end (graph created from the same host arrays
+ run + result to host + destroy) and with ours device-resident.

  python tools/golden_gpu.py [--out profiles/golden_gpu_r01.json] [--bc-sources 2]
"""
import argparse
import ctypes as C
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2401_02472_b200 as gdx  # noqa: E402

LIB = os.path.join(ROOT, "oracle", "_ref", "libgolden.so")
I32 = C.POINTER(C.c_int32)


def ptr(a):
    return a.ctypes.data_as(I32) if a is not None else None


def csr_args(h, weights=True):
    w = h.weights if weights else None
    return [h.n, h.m, ptr(h.offsets), ptr(h.dests), ptr(w), ptr(h.rev_offsets), ptr(h.rev_srcs),
            ptr(h.rev_eid)]


def wall(fn, reps):
    fn()
    t = []
    for _ in range(reps):
        t0 = time.perf_counter()
        r = fn()
        t.append(time.perf_counter() - t0)
    return min(t), r


def ours_e2e(h, run, keys):
    """create from the host arrays the algorithm needs (what the golden unit
    uploads), run, result to host, destroy."""
    view = gdx.HostCsr(h.n, h.m, h.directed, *[getattr(h, k) if k in keys else None for k in
                                                ("offsets", "dests", "weights", "rev_offsets",
                                                 "rev_srcs", "rev_eid")])
    g = gdx.DeviceGraph.from_csr(view)
    try:
        return run(g)
    finally:
        g.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--bc-sources", type=int, default=2)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--skip", default="C5", help="comma list of pr,C1,C5,tc,bc to skip")
    a = ap.parse_args()
    L = C.CDLL(LIB)
    L.golden_tc.restype = C.c_longlong
    res = {}

    # C2 PageRank RMAT-24
    if "pr" not in a.skip:
        dg = gdx.DeviceGraph.generate("rmat", 1 << 24, 1 << 28, seed=1, directed=True)
        h = dg.download()
        rank_g = np.empty(h.n, np.float64)
        tg, _ = wall(lambda: L.golden_pr(*csr_args(h), C.c_double(0.85), C.c_double(1e-6), 100,
                                         rank_g.ctypes.data_as(C.POINTER(C.c_double))), a.reps)
        t_dev, (r_ours, rounds) = wall(lambda: dg.pagerank(0.85, 1e-6, 100), a.reps)
        t_e2e, _ = wall(lambda: ours_e2e(h, lambda g: g.pagerank(0.85, 1e-6, 100),
                                          ("offsets", "rev_offsets", "rev_srcs")), a.reps)
        rel = float(np.max(np.abs(r_ours - rank_g) / np.abs(rank_g)))
        res["C2_pagerank_rmat24"] = {"m": h.m, "rounds": rounds, "golden_s": tg, "ours_e2e_s": t_e2e,
                                     "ours_resident_s": t_dev, "max_rel_diff": rel,
                                     "golden_gteps": h.m * rounds / tg / 1e9,
                                     "ours_e2e_gteps": h.m * rounds / t_e2e / 1e9}
        print(json.dumps(res["C2_pagerank_rmat24"]), flush=True)
        dg.close()

    # C1 SSSP RMAT-18 (and C5 RMAT-26)
    for key, sc in (("C1_sssp_rmat18", 18), ("C5_sssp_rmat26", 26)):
        if key.split("_")[0] in a.skip:
            continue
        dg = gdx.DeviceGraph.generate("rmat", 1 << sc, 16 << sc, seed=1, directed=False,
                                      weights=(1, 100))
        h = dg.download()
        dist_g = np.empty(h.n, np.int32)
        tg, _ = wall(lambda: L.golden_sssp(*csr_args(h), 0, ptr(dist_g)), 1 if sc > 20 else a.reps)
        t_dev, d_ours = wall(lambda: dg.sssp(0), a.reps)
        t_e2e, _ = wall(lambda: ours_e2e(h, lambda g: g.sssp(0), ("offsets", "dests", "weights")),
                        1 if sc > 20 else a.reps)
        inf32 = np.iinfo(np.int32).max // 2
        same = bool(np.array_equal(np.where(dist_g >= inf32, -1, dist_g),
                                   np.where(d_ours >= (2**63 - 1) // 2, -1, d_ours)))
        res[key] = {"m": h.m, "golden_s": tg, "ours_e2e_s": t_e2e, "ours_resident_s": t_dev,
                    "identical": same, "golden_gteps": h.m / tg / 1e9,
                    "ours_e2e_gteps": h.m / t_e2e / 1e9}
        print(key, json.dumps(res[key]), flush=True)
        dg.close()
        del h

    # C3 TC uniform 2^24
    if "tc" not in a.skip:
        dg = gdx.DeviceGraph.generate("uniform", 1 << 24, 1 << 27, seed=1, directed=False)
        h = dg.download()
        tg, cg = wall(lambda: L.golden_tc(*csr_args(h, weights=False)), 1)
        t_dev, c_ours = wall(lambda: dg.tc(), a.reps)
        t_e2e, _ = wall(lambda: ours_e2e(h, lambda g: g.tc(), ("offsets", "dests")), a.reps)
        res["C3_tc_uniform24"] = {"m": h.m, "golden_s": tg, "ours_e2e_s": t_e2e,
                                  "ours_resident_s": t_dev, "golden_count": int(cg),
                                  "ours_count": int(c_ours), "golden_gteps": h.m / tg / 1e9,
                                  "ours_e2e_gteps": h.m / t_e2e / 1e9}
        print(json.dumps(res["C3_tc_uniform24"]), flush=True)
        dg.close()

    # C4 BC grid (a few sources: the golden path takes a host round trip per level)
    if "bc" not in a.skip:
        dg = gdx.DeviceGraph.generate("grid", 4899, seed=1, keep=0.55, directed=False)
        h = dg.download()
        deg = np.diff(h.offsets)
        src = sorted(np.random.default_rng(1).choice(np.flatnonzero(deg > 0), a.bc_sources,
                                                     replace=False).tolist())
        s32 = np.asarray(src, np.int32)
        bc_g = np.empty(h.n, np.float64)
        tg, _ = wall(lambda: L.golden_bc(*csr_args(h, weights=False), ptr(s32), len(src),
                                         bc_g.ctypes.data_as(C.POINTER(C.c_double))), 1)
        t_dev, b_ours = wall(lambda: dg.bc(src), 1)
        t_e2e, _ = wall(lambda: ours_e2e(h, lambda g: g.bc(src), ("offsets", "dests")), 1)
        fin = np.isfinite(bc_g)
        rel = float(np.max(np.abs(b_ours[fin] - bc_g[fin]) / np.maximum(np.abs(bc_g[fin]), 1e-12)))
        res["C4_bc_grid4899"] = {"m": h.m, "sources": len(src), "golden_s": tg, "ours_e2e_s": t_e2e,
                                 "ours_resident_s": t_dev, "max_rel_diff_where_golden_finite": rel,
                                 "golden_nonfinite": int((~fin).sum()),
                                 "golden_gteps": h.m * len(src) / tg / 1e9,
                                 "ours_e2e_gteps": h.m * len(src) / t_e2e / 1e9}
        print(json.dumps(res["C4_bc_grid4899"]), flush=True)
        dg.close()
    if a.out:
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
