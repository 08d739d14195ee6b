"""Generate the committed golden vectors from the REFERENCE ITSELF.

Runs in the build container only (needs oracle/_ref/libgraphdsl_ref.so, which
`make -C oracle ref` compiles from /root/reference/proj/core/src).  Every
expected value below is produced by the reference's own code:

* graphs: graphdsl::genUniformEdges / genRmatEdges, CsrGraph::buildFromEdges,
  CsrGraph::withRandomWeights;
* results: interp::run on the corpus programs (sequential mode) and the
  textbook oracles::sssp / pr / bc / tc / bfsLevels.

Outputs (committed): tests/golden/known.json (hand-checkable fixtures from the
reference tests) and tests/golden/sweep.npz (acceptance criterion 2:
acceptance_main.cpp:108-181, 200 seeds, makeGraph :62-67).

usage: python tests/golden/make_golden.py
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

from oracle import Ref  # noqa: E402


def csr_dict(g) -> dict:
    h = g.host()
    return {"n": h.n, "m": h.m, "directed": h.directed, "offsets": h.offsets.tolist(),
            "dests": h.dests.tolist(), "weights": h.weights.tolist(),
            "rev_offsets": h.rev_offsets.tolist(), "rev_srcs": h.rev_srcs.tolist(),
            "rev_eid": h.rev_eid.tolist()}


def known(ref: Ref) -> dict:
    cases = {}

    def add(name, g, **res):
        cases[name] = {"graph": csr_dict(g), **res}

    # test_oracles.cpp:26 / test_interpreter.cpp:46-52 -- TC(K4) = 4
    k4u, k4v = zip(*[(u, v) for u in range(4) for v in range(u + 1, 4)])
    k4 = ref.build(4, k4u, k4v, None, False)
    add("k4", k4, tc=k4.interp_tc()[0], tc_oracle=k4.oracle_tc(),
        sssp0=k4.interp_sssp(0)[0].tolist())
    # test_interpreter.cpp:34-44 -- weighted triangle [0, 5, 6]
    tri = ref.build(3, [0, 1, 0], [1, 2, 2], [5, 1, 7], False)
    d, mod, fin = tri.interp_sssp(0)
    add("weighted_triangle", tri, sssp0=d.tolist(), modified=mod.tolist(), finished=fin,
        bc_all=tri.interp_bc([0, 1, 2]).tolist(), tc=tri.interp_tc()[0])
    # test_oracles.cpp:41-48 -- unreachable node keeps INF
    tri4 = ref.build(4, [0, 1, 0], [1, 2, 2], [5, 1, 7], False)
    add("weighted_triangle_isolated", tri4, sssp0=tri4.interp_sssp(0)[0].tolist(),
        sssp0_oracle=tri4.oracle_sssp(0).tolist())
    # test_interpreter.cpp:54-62 -- BC(path3) = [0, 2, 0]
    p3 = ref.build(3, [0, 1], [1, 2], None, False)
    add("path3", p3, bc_all=p3.interp_bc([0, 1, 2]).tolist(),
        bc_oracle=p3.oracle_bc([0, 1, 2]).tolist())
    # test_oracles.cpp:67-76 -- 7-cycle: equal scores
    c7 = ref.build(7, list(range(7)), [(v + 1) % 7 for v in range(7)], None, False)
    add("cycle7", c7, bc_all=c7.interp_bc(list(range(7))).tolist())
    # test_interpreter.cpp:64-72 -- PR 2-cycle = [0.5, 0.5]
    cyc = ref.build(2, [0, 1], [1, 0], None, True)
    r, it = cyc.interp_pr(0.85, 1e-9, 110)
    add("pr_two_cycle", cyc, pr=r.tolist(), pr_iter=it)
    # test_oracles.cpp:85-92 -- PR sums to one (dangling mass redistributed)
    eu, ev = ref.gen_rmat_edges(40, 100, 23)
    g40 = ref.build(40, eu, ev, None, True)
    r, it = g40.interp_pr(0.85, 1e-12, 1000)
    add("pr_rmat40", g40, pr=r.tolist(), pr_iter=it,
        pr_oracle=g40.oracle_pr(0.85, 1e-12, 1000).tolist())
    # pr.sp:25 -- maxIter=3 runs 4 rounds == oracles::pr(..., 4)
    r, it = g40.interp_pr(0.85, 0.0, 3)
    add("pr_maxiter3", g40, pr=r.tolist(), pr_iter=it,
        pr_oracle4=g40.oracle_pr(0.85, 0.0, 4).tolist())
    # test_csr.cpp:28-38 -- directed triangle; :67-71 duplicates keep min weight
    dt = ref.build(3, [0, 0, 1], [1, 2, 2], None, True)
    add("directed_triangle", dt)
    dup = ref.build(2, [0, 0, 0], [1, 1, 1], [9, 4, 6], True)
    add("dup_min_weight", dup)
    # self loops stored once (csr.cpp:43), isolated nodes, unsorted input
    sl = ref.build(5, [3, 0, 2, 2, 4, 1], [3, 4, 0, 2, 1, 4], [2, 7, 3, 1, 9, 4], False)
    add("self_loops", sl, sssp0=sl.interp_sssp(0)[0].tolist(), tc=sl.interp_tc()[0],
        bc_all=sl.interp_bc(list(range(5))).tolist())
    # interpreter-level error behaviour
    cases["errors"] = {
        "sssp_src_out_of_range": _err(lambda: tri.interp_sssp(99)),
        "bc_source_out_of_range": _err(lambda: tri.interp_bc([0, 7])),
        "invalid_edge": _err(lambda: ref.build(2, [0], [5], None, True)),
        "negative_weight": _err(lambda: ref.build(2, [0], [1], [-3], True)),
    }
    return cases


def _err(fn) -> str:
    try:
        fn()
    except Exception as e:  # OracleError carries "<Kind>: <message>"
        return str(e)
    return ""


def make_graph(ref: Ref, seed: int, max_nodes: int, directed: bool):
    """acceptance_main.cpp:62-67"""
    n = 2 + seed % (max_nodes - 1)
    m = n * (2 + seed % 3)
    if seed % 2 == 0:
        u, v = ref.gen_uniform_edges(n, m, seed)
    else:
        u, v = ref.gen_rmat_edges(n, m, seed)
    return ref.build(n, u, v, None, directed)


def sweep(ref: Ref) -> dict:
    out = {}
    for seed in range(1, 201):
        und = make_graph(ref, seed, 60, False).with_random_weights(1, 100, seed)
        dr = make_graph(ref, seed, 60, True)
        n = und.n
        src = seed % n
        hu, hd = und.host(), dr.host()
        p = f"s{seed}_"
        for k in ("offsets", "dests", "weights"):
            out[p + "und_" + k] = getattr(hu, k)
            out[p + "dir_" + k] = getattr(hd, k)
        out[p + "n"] = np.array([n, hu.m, hd.m])
        dist, mod, fin = und.interp_sssp(src)
        out[p + "sssp"] = dist
        assert not mod.any() and fin
        out[p + "tc"] = np.array([und.interp_tc()[0], und.oracle_tc()])
        out[p + "bc"] = und.interp_bc(list(range(n)))
        out[p + "bc_oracle"] = und.oracle_bc(list(range(n)))
        r, it = dr.interp_pr(0.85, 1e-9, 110)
        out[p + "pr"] = r
        out[p + "pr_iter"] = np.array([it])
        out[p + "pr_oracle"] = dr.oracle_pr(0.85, 1e-9, 110)
    return out


def main() -> None:
    ref = Ref()
    with open(os.path.join(HERE, "known.json"), "w") as f:
        json.dump(known(ref), f, indent=0, sort_keys=True)
    np.savez_compressed(os.path.join(HERE, "sweep.npz"), **sweep(ref))
    print("wrote known.json and sweep.npz")


if __name__ == "__main__":
    main()
