"""GPU parity: the B200 kernels (through the C ABI) against the oracle.

Bars (north star): SSSP distances and triangle counts bit-exact; PageRank and
BC within 1e-6 relative (tightened to 1e-9 on small graphs, where the only
difference is floating-point summation order), PageRank with the same number
of fixedPoint rounds as the reference.
"""
from __future__ import annotations

import numpy as np
import pytest

from conftest import G, ROOT, known_graph, rel_err, reverse_of, sweep_graphs

pytestmark = pytest.mark.gpu
INF = (2**63 - 1) // 2
CSR_KEYS = ("offsets", "dests", "weights", "rev_offsets", "rev_srcs", "rev_eid")


def upload(gdx, g, with_rev=True):
    if not with_rev:
        g = G(g.n, g.m, g.directed, g.offsets, g.dests, g.weights)
    return gdx.DeviceGraph.from_csr(g)


def assert_same_csr(dev_host, exp, keys=CSR_KEYS):
    for k in keys:
        a, b = np.asarray(getattr(dev_host, k)), np.asarray(getattr(exp, k))
        assert np.array_equal(a, b), k


# ---- hand-checkable fixtures (reference tests) ---------------------------------

def test_known_fixtures(gdx, known):
    r = gdx.run("ComputeSSSP", known_graph(known["weighted_triangle"]), {"src": 0})
    assert list(r.property("dist")) == [0, 5, 6]
    assert not r.property("modified").any() and r.scalar("finished") is True
    c = known["weighted_triangle_isolated"]
    assert list(gdx.run("sssp", known_graph(c), {"src": 0}).property("dist")) == c["sssp0"]
    r = gdx.run("ComputeTC", known_graph(known["k4"]), {})
    assert r.scalar("triangleCount") == 4 and r.return_value == 4
    r = gdx.run("ComputeBC", known_graph(known["path3"]), {"sourceSet": [0, 1, 2]})
    assert list(r.property("bc")) == [0.0, 2.0, 0.0]
    c = known["cycle7"]
    bc = gdx.run("bc", known_graph(c), {"sourceSet": list(range(7))}).property("bc")
    assert rel_err(bc, c["bc_all"]) < 1e-12
    c = known["pr_two_cycle"]
    r = gdx.run("ComputePR", known_graph(c), {"damping": 0.85, "threshold": 1e-9, "maxIter": 110})
    assert rel_err(r.property("rank"), c["pr"]) < 1e-12 and r.scalar("iter") == c["pr_iter"]
    for name, thr, mi in (("pr_rmat40", 1e-12, 1000), ("pr_maxiter3", 0.0, 3)):
        c = known[name]
        r = gdx.run("pr", known_graph(c), {"damping": 0.85, "threshold": thr, "maxIter": mi})
        assert r.scalar("iter") == c["pr_iter"], name
        assert rel_err(r.property("rank"), c["pr"]) < 1e-12, name
    c = known["self_loops"]
    g = known_graph(c)
    assert list(gdx.run("sssp", g, {"src": 0}).property("dist")) == c["sssp0"]
    assert gdx.run("tc", g, {}).return_value == c["tc"]
    assert rel_err(gdx.run("bc", g, {"sourceSet": list(range(5))}).property("bc"), c["bc_all"]) < 1e-12


def test_errors_match_reference(gdx, known):
    err = known["errors"]
    g = known_graph(known["weighted_triangle"])
    dg = gdx.DeviceGraph.from_csr(g)
    with pytest.raises(gdx.GraphdslError) as e:
        dg.sssp(99)
    assert str(e.value) == err["sssp_src_out_of_range"] and e.value.kind == "RuntimeError"
    with pytest.raises(gdx.GraphdslError) as e:
        dg.bc([0, 7])
    assert str(e.value) == err["bc_source_out_of_range"]
    with pytest.raises(gdx.GraphdslError) as e:
        gdx.DeviceGraph.build_from_edges(2, [0], [5], None, True)
    assert str(e.value) == err["invalid_edge"] and e.value.kind == "InvalidEdge"
    with pytest.raises(gdx.GraphdslError) as e:
        gdx.DeviceGraph.build_from_edges(2, [0], [1], [-3], True)
    assert str(e.value) == err["negative_weight"]
    # first offending edge in input order decides (csr.cpp:29-40)
    with pytest.raises(gdx.GraphdslError, match=r"NegativeWeight: edge \(0, 1\)"):
        gdx.DeviceGraph.build_from_edges(3, [0, 0], [1, 9], [-1, 1], True)
    # pr.sp:9 divides by numNodes; interp raises on an empty graph
    empty = gdx.DeviceGraph.build_from_edges(0, [], [], None, True)
    with pytest.raises(gdx.GraphdslError, match="division by zero"):
        empty.pagerank()
    assert empty.tc() == 0
    # fixedPoint cap 10n+100 (interpreter.cpp:977-986): never-settling PR
    two = gdx.DeviceGraph.build_from_edges(2, [0, 1], [1, 0], None, True)
    with pytest.raises(gdx.GraphdslError) as e:
        two.pagerank(0.85, -1.0, 1000)
    assert e.value.kind == "NonTermination"
    r, it = two.pagerank(0.85, -1.0, 50)  # settles by maxIter: 51 rounds <= cap
    assert it == 51


def test_shard_entry_points_validate(gdx, known):
    """The multi-GPU entry points fail loudly on misuse instead of launching."""
    import torch
    g = known_graph(known["weighted_triangle"])
    dg = gdx.DeviceGraph.from_csr(g)
    d = torch.zeros(dg.n, dtype=torch.int32, device="cuda")
    with pytest.raises(gdx.GraphdslError, match="no shard plan"):
        dg.sssp_shard_relax32_delta(d, d.clone(), d.clone())
    with pytest.raises(gdx.GraphdslError, match="no shard plan"):
        dg.sssp_shard_frontier32(d, d.clone())
    with pytest.raises(gdx.GraphdslError, match="out of bounds"):
        dg.sssp_shard_setup(0, dg.n + 1)
    with pytest.raises(gdx.GraphdslError, match="no p2p plan"):
        dg.pr_p2p_rounds(0, 4, 0.85, 1e-6, 100, 0.0)
    dg.sssp_shard_apply32(d, d, d, 0)  # nothing to apply: a no-op


# ---- acceptance criterion 2 sweep: 200 reference graphs ------------------------------

def test_sweep_vs_reference(gdx, sweep):
    for seed in range(1, 201):
        und, dr = sweep_graphs(sweep, seed)
        p = f"s{seed}_"
        n = und.n
        du = upload(gdx, und, with_rev=(seed % 2 == 0))  # odd seeds: reverse CSR built on GPU
        if seed % 2:
            assert_same_csr(du.download(), und, ("rev_offsets", "rev_srcs", "rev_eid"))
        assert np.array_equal(du.sssp(seed % n), sweep[p + "sssp"]), seed
        assert du.tc() == int(sweep[p + "tc"][0]), seed
        assert rel_err(du.bc(list(range(n))), sweep[p + "bc"]) < 1e-9, seed
        dd = upload(gdx, dr)
        r, it = dd.pagerank(0.85, 1e-9, 110)
        assert it == int(sweep[p + "pr_iter"][0]), seed
        assert rel_err(r, sweep[p + "pr"]) < 1e-9, seed
        du.close()
        dd.close()


# ---- GPU CSR builder == CsrGraph::buildFromEdges -------------------------------------

@pytest.mark.parametrize("n,m,directed,weighted,seed", [
    (1, 0, True, False, 1), (5, 0, False, False, 1), (50, 400, False, True, 2),
    (300, 5000, True, True, 3), (1 << 12, 1 << 16, False, False, 4),
    (1 << 14, 1 << 17, True, True, 5), (70000, 300000, False, True, 6)])
def test_gpu_builder_bit_exact(gdx, port, n, m, directed, weighted, seed):
    rng = np.random.default_rng(seed)
    u, v = port.gen_rmat_edges(n, m, seed) if m else (np.zeros(0, np.int32),) * 2
    w = rng.integers(0, 50, size=m).astype(np.int32) if weighted else None
    exp = port.build_from_edges(n, u, v, w, directed)
    dg = gdx.DeviceGraph.build_from_edges(n, u, v, w, directed)
    assert (dg.n, dg.m, dg.directed) == (exp.n, exp.m, exp.directed)
    assert_same_csr(dg.download(), exp)


def test_gpu_builder_c1_reference_graph(gdx, port):
    """C1 input exactly as the reference builds it: genRmatEdges(2^18, 2^22, 1)."""
    u, v = port.gen_rmat_edges(1 << 18, 1 << 22, 1)
    exp = port.build_from_edges(1 << 18, u, v, None, False)
    assert exp.m == 7611081
    dg = gdx.DeviceGraph.build_from_edges(1 << 18, u, v, None, False)
    assert_same_csr(dg.download(), exp, ("offsets", "dests", "rev_offsets", "rev_srcs", "rev_eid"))


# ---- SSSP ----------------------------------------------------------------------------

def test_sssp_c1_bit_exact(gdx, port):
    """Config 1: RMAT-18, ef 16, undirected, weights U[1,100] (withRandomWeights)."""
    u, v = port.gen_rmat_edges(1 << 18, 1 << 22, 1)
    g = port.with_random_weights(port.build_from_edges(1 << 18, u, v, None, False), 1, 100, 1)
    dg = gdx.DeviceGraph.from_csr(g)
    for src in (0, 1, 12345, 262143):
        st = {}
        got = dg.sssp(src, stats=st)
        exp = port.sssp(g, src)
        assert np.array_equal(got, exp), src
        if src == 0:
            assert (exp < INF).sum() == 174054 and exp[exp < INF].max() == 209
            assert st["rounds"] >= 2 and st["edges_visited"] >= g.m * 0.5


@pytest.mark.parametrize("mode", ["persistent", "scan", "graph", "scan_split", "graph_split"])
def test_sssp_modes_c1(gdx, port, mode, monkeypatch):
    """Both SSSP executions (persistent cooperative kernel for small graphs,
    frontier-scan rounds for large ones) are bit-exact on config 1; *_split:
    the large-graph form with small vertices (<= 8 edges) in their own queue."""
    monkeypatch.setenv("GDX_SSSP_MODE", mode.split("_")[0])
    monkeypatch.setenv("GDX_SSSP_SPLIT", "1" if mode.endswith("split") else "0")
    u, v = port.gen_rmat_edges(1 << 18, 1 << 22, 1)
    g = port.with_random_weights(port.build_from_edges(1 << 18, u, v, None, False), 1, 100, 1)
    dg = gdx.DeviceGraph.from_csr(g)
    for src in (0, 262143):
        assert np.array_equal(dg.sssp(src), port.sssp(g, src)), src


@pytest.mark.parametrize("mode", ["persistent", "scan", "graph"])
def test_sssp_64bit_distances(gdx, port, mode, monkeypatch):
    monkeypatch.setenv("GDX_SSSP_MODE", mode)
    u, v = port.gen_rmat_edges(5000, 40000, 8)
    g = port.build_from_edges(5000, u, v, None, True)
    g.weights = np.random.default_rng(1).integers(1 << 28, 1 << 30, size=g.m).astype(np.int32)
    dg = gdx.DeviceGraph.from_csr(g)
    for src in (0, 17):
        assert np.array_equal(dg.sssp(src), port.sssp(g, src))


@pytest.mark.parametrize("weights", [(1, 100), (300, 600)])
def test_sssp_16bit_first_attempt(gdx, port, weights, monkeypatch):
    """Large graphs try 16-bit distances first (GDX_SSSP_NARROW=1 forces it
    here): exact when they fit (C1's weights, max distance 209), and an
    overflow (a 100x100 grid with weights 300..600 reaches ~10^5) reruns the
    call at 32 bits -- on this handle and on the next call too."""
    monkeypatch.setenv("GDX_SSSP_NARROW", "1")
    gu, gv = port.gen_grid_ctr(100, 2.0, 1)
    g = port.build_from_edges(100 * 100, gu, gv, None, False)
    g.weights = np.random.default_rng(3).integers(*weights, size=g.m).astype(np.int32)
    dg = gdx.DeviceGraph.from_csr(g)
    for mode in ("graph", "scan"):
        monkeypatch.setenv("GDX_SSSP_MODE", mode)
        for src in (0, 5050, 0):
            exp = port.sssp(g, src)
            assert np.array_equal(dg.sssp(src), exp), (mode, src)
    assert (exp[exp < INF].max() > 65535) == (weights[0] == 300)


def test_sssp_zero_weights_and_unreachable(gdx, port):
    u, v = port.gen_uniform_edges(3000, 9000, 4)
    g = port.build_from_edges(3000, u, v, None, True)
    g.weights = (np.arange(g.m) % 3).astype(np.int32)  # many zero-weight edges
    dg = gdx.DeviceGraph.from_csr(g)
    got = dg.sssp(0)
    assert np.array_equal(got, port.sssp(g, 0))
    assert (got == INF).any()


def test_sssp_device_output(gdx, port):
    torch = pytest.importorskip("torch")
    u, v = port.gen_rmat_edges(1 << 12, 1 << 15, 3)
    g = port.with_random_weights(port.build_from_edges(1 << 12, u, v, None, False), 1, 100, 3)
    dg = gdx.DeviceGraph.from_csr(g)
    out = torch.empty(g.n, dtype=torch.int64, device="cuda")
    dg.sssp(5, out=out)
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), port.sssp(g, 5))


# ---- PageRank ----------------------------------------------------------------------

@pytest.mark.parametrize("scale,directed", [(10, True), (16, True), (16, False), (18, True)])
def test_pagerank_rmat(gdx, port, scale, directed):
    n = 1 << scale
    u, v = port.gen_rmat_edges(n, 16 * n, scale)
    g = port.build_from_edges(n, u, v, None, directed)
    dg = gdx.DeviceGraph.from_csr(g)
    for thr, mi in ((1e-6, 100), (1e-9, 110), (0.0, 5)):
        exp, it = port.pr(g, 0.85, thr, mi)
        got, rounds = dg.pagerank(0.85, thr, mi)
        assert rounds == it, (thr, mi)
        assert rel_err(got, exp) < 1e-9, (thr, mi)


def test_pagerank_hub_rows_span_tiles(gdx, port):
    """A star with in-degree >> tile size exercises the cross-tile slot path."""
    n = 20000
    u = np.arange(1, n, dtype=np.int32)
    v = np.zeros(n - 1, np.int32)
    u2, v2 = port.gen_uniform_edges(n, 5 * n, 9)
    g = port.build_from_edges(n, np.concatenate([u, u2]), np.concatenate([v, v2]), None, True)
    dg = gdx.DeviceGraph.from_csr(g)
    exp, it = port.pr(g, 0.85, 1e-10, 200)
    got, rounds = dg.pagerank(0.85, 1e-10, 200)
    assert rounds == it and rel_err(got, exp) < 1e-9


def test_pagerank_isolated_and_dangling(gdx, port):
    g = port.build_from_edges(10, [0, 1, 2, 2], [1, 2, 0, 3], None, True)
    exp, it = port.pr(g, 0.85, 1e-12, 500)
    got, rounds = gdx.DeviceGraph.from_csr(g).pagerank(0.85, 1e-12, 500)
    assert rounds == it and rel_err(got, exp) < 1e-12
    assert abs(got.sum() - 1.0) < 1e-9


# ---- Triangle counting ---------------------------------------------------------------

@pytest.mark.parametrize("kind,scale,directed", [("uniform", 16, False), ("rmat", 14, False),
                                                 ("rmat", 14, True), ("uniform", 18, True)])
def test_tc(gdx, port, kind, scale, directed):
    n = 1 << scale
    u, v = (port.gen_uniform_edges if kind == "uniform" else port.gen_rmat_edges)(n, 8 * n, scale)
    g = port.build_from_edges(n, u, v, None, directed)
    dg = gdx.DeviceGraph.from_csr(g)
    exp = port.tc(g)
    assert dg.tc() == exp
    mid = n // 3
    assert dg.tc_range(0, mid) + dg.tc_range(mid, n) == exp
    assert dg.tc_range(mid, n) == port.tc_range(g, mid, n)


# ---- Betweenness centrality ------------------------------------------------------------

@pytest.fixture(params=["grid", "cta", "cta1", "cta2", "cta_nokids"])
def bc_mode(request, monkeypatch):
    """Both BC executions: grid-wide level-synchronous kernels, and one CTA
    cluster per source (the default once there are >= max(16, #SM/4) sources)
    with the cluster size picked from the SM count, or forced to 1 / 2; and the
    CTA kernel's backward pass scanning the adjacency instead of the children
    recorded by the forward pass (GDX_BC_KIDS=0)."""
    mode = request.param
    monkeypatch.setenv("GDX_BC_MODE", "grid" if mode == "grid" else "cta")
    if mode in ("cta1", "cta2"):
        monkeypatch.setenv("GDX_BC_CLUSTER", mode[-1])
    if mode == "cta_nokids":
        monkeypatch.setenv("GDX_BC_KIDS", "0")
    return mode


def test_bc_rmat(gdx, port, bc_mode):
    n = 1 << 12
    u, v = port.gen_rmat_edges(n, 8 * n, 21)
    for directed in (False, True):
        g = port.build_from_edges(n, u, v, None, directed)
        dg = gdx.DeviceGraph.from_csr(g)
        srcs = [0, 1, 2, 5, 77, 1000, 4095, 1]  # duplicates are legal
        assert rel_err(dg.bc(srcs), port.bc(g, srcs)) < 1e-9, directed


def test_bc_grid_and_overflow(gdx, port, bc_mode):
    gu, gv = port.gen_grid_ctr(100, 0.55, 3)
    g = port.build_from_edges(100 * 100, gu, gv, None, False)
    srcs = [0, 4242, 9999, 5050]
    assert rel_err(gdx.DeviceGraph.from_csr(g).bc(srcs), port.bc(g, srcs)) < 1e-9
    side = 600  # full grid: the reference's double sigma overflows
    gu, gv = port.gen_grid_ctr(side, 2.0, 1)
    g = port.build_from_edges(side * side, gu, gv, None, False)
    got = gdx.DeviceGraph.from_csr(g).bc([0])
    assert np.isfinite(got).all()
    assert rel_err(got, port.bc(g, [0])) < 1e-6


def test_bc_many_sources_slot_reuse(gdx, port):
    """More sources than CTAs: the default picks CTA mode and every CTA slot is
    reused for several sources (its level tags advance in between)."""
    gu, gv = port.gen_grid_ctr(60, 0.6, 5)
    g = port.build_from_edges(3600, gu, gv, None, False)
    srcs = list(range(0, 3600, 11))  # 328 sources > #SM
    dg = gdx.DeviceGraph.from_csr(g)
    st = {}
    got = dg.bc(srcs, stats=st)
    assert st["launches"] == 2  # one k_bc_cta launch + the ordered slot sum
    assert rel_err(got, port.bc(g, srcs)) < 1e-9


@pytest.mark.parametrize("mode", ["grid", "cta"])
def test_bc_and_pr_reproducible(gdx, port, mode, monkeypatch):
    """No floating-point atomics on the score paths: BC sums the per-slot
    (CTA mode) or per-source (grid mode) partials in a fixed order, PageRank
    sums rows by chunk partials -- repeated calls give bit-identical results."""
    monkeypatch.setenv("GDX_BC_MODE", mode)
    n = 1 << 13
    u, v = port.gen_rmat_edges(n, 16 * n, 4)
    g = port.build_from_edges(n, u, v, None, False)
    dg = gdx.DeviceGraph.from_csr(g)
    srcs = list(range(0, n, 97))
    first = dg.bc(srcs)
    for _ in range(3):
        assert np.array_equal(dg.bc(srcs), first)
    assert rel_err(first, port.bc(g, srcs)) < 1e-9
    d = gdx.DeviceGraph.from_csr(port.build_from_edges(n, u, v, None, True))
    r0, it0 = d.pagerank(0.85, 1e-9, 100)
    for _ in range(3):
        r, it = d.pagerank(0.85, 1e-9, 100)
        assert it == it0 and np.array_equal(r, r0)


def test_bc_level_tags_run_out(gdx, port, monkeypatch):
    """Level tags: a slot's sources use increasing tag ranges (no per-source
    restore); when the tags would pass INT32_MAX the slot is cleared.  Start the
    tags just below that limit so the clearing runs inside a call and between
    calls on the same handle."""
    gu, gv = port.gen_grid_ctr(60, 0.6, 5)
    g = port.build_from_edges(3600, gu, gv, None, False)
    monkeypatch.setenv("GDX_BC_MODE", "cta")
    monkeypatch.setenv("GDX_BC_TAG_START", str(2**31 - 1 - 3602 - 300))
    srcs = list(range(0, 3600, 11))  # several sources per slot
    dg = gdx.DeviceGraph.from_csr(g)
    exp = port.bc(g, srcs)
    for _ in range(3):
        assert rel_err(dg.bc(srcs), exp) < 1e-9


# ---- GPU generators == their CPU twin ---------------------------------------------------

def test_generators_match_cpu_twin(gdx, port):
    n, E = 1 << 14, 1 << 17
    dg = gdx.DeviceGraph.generate("rmat", n, E, seed=5, directed=True)
    u, v = port.gen_rmat_ctr(n, E, 5)
    assert_same_csr(dg.download(), port.build_from_edges(n, u, v, None, True),
                    ("offsets", "dests", "rev_offsets", "rev_srcs", "rev_eid"))
    dg = gdx.DeviceGraph.generate("uniform", 5000, 40000, seed=6, directed=False,
                                  weights=(1, 100))
    u, v = port.gen_uniform_ctr(5000, 40000, 6)
    exp = port.build_from_edges(5000, u, v, None, False)
    exp.weights = port.hash_weights(exp, 1, 100, 6)
    assert_same_csr(dg.download(), exp)
    dg = gdx.DeviceGraph.generate("grid", 64, seed=7, keep=0.55, directed=False)
    u, v = port.gen_grid_ctr(64, 0.55, 7)
    assert_same_csr(dg.download(), port.build_from_edges(64 * 64, u, v, None, False),
                    ("offsets", "dests", "rev_offsets", "rev_srcs", "rev_eid"))


# ---- the C++ drop-in (include/gdx_graphdsl.hpp) against interp::run itself ----------------

def test_cpp_dropin_against_interp(gdx):
    import os
    import subprocess
    from conftest import ROOT
    exe = os.path.join(ROOT, "oracle", "_ref", "gdx_dropin_test")
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref/gdx_dropin_test not built (needs /root/reference at build time)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "DROPIN PASS" in r.stdout, r.stdout + r.stderr


@pytest.mark.parametrize("stage", ["0", "7"])
def test_sssp_warp_chunk_queue(gdx, port, stage, monkeypatch):
    """Large frontiers overflow the block staging into per-warp chunks of the
    global queue (padded with sentinel items); force that path on C1-sized
    graphs (GDX_SSSP_STAGE caps the staging) and check bit-exactness."""
    monkeypatch.setenv("GDX_SSSP_STAGE", stage)
    u, v = port.gen_rmat_edges(1 << 16, 1 << 20, 5)
    g = port.with_random_weights(port.build_from_edges(1 << 16, u, v, None, False), 1, 100, 5)
    dg = gdx.DeviceGraph.from_csr(g)
    for src in (0, 999):
        assert np.array_equal(dg.sssp(src), port.sssp(g, src)), src


# ---- multi-GPU shards through the real kernels ------------------------------------------

def _gpu_shard_worker(rank, world, port, q):
    import os
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK="0")
    import torch.distributed as tdist
    import paper_2401_02472_b200 as G
    from paper_2401_02472_b200 import distributed as D
    from oracle import Port
    # every rank shares cuda:0, so the collectives go over gloo (CPU-staged);
    # on the GPU box's multi-GPU runs the same code uses NCCL on device tensors
    D.init_from_env("gloo")
    p = Port()
    n = 1 << 12
    u, v = p.gen_rmat_edges(n, 16 * n, 21)
    gd = p.build_from_edges(n, u, v, None, True)
    gu = p.with_random_weights(p.build_from_edges(n, u, v, None, False), 1, 100, 21)
    exd = D.DeviceExecutor(G.DeviceGraph.from_csr(gd))
    r, rounds = D.sharded_pr(exd, 0.85, 1e-9, 110)
    # the peer-memory exchange (CUDA IPC between the ranks' processes), twice:
    # the second call reuses the exported blocks (publish parity carries over)
    r2, rounds2 = D.sharded_pr_p2p(exd, 0.85, 1e-9, 110)
    r3, rounds3 = D.sharded_pr_p2p(exd, 0.85, 1e-9, 110)
    exu = D.DeviceExecutor(G.DeviceGraph.from_csr(gu))
    st32, st64, stb = {}, {}, {}
    d = D.sharded_sssp(exu, 7, stats=st32)  # int32 replicas
    d64 = D.sharded_sssp(exu, 7, width=64, stats=st64)
    dd = D.sharded_sssp(exu, 7, exchange="dense")
    # weights near 2^30: the int32 rounds overflow and the call reruns over int64
    gb = p.with_random_weights(p.build_from_edges(n, u, v, None, False), 1 << 29, 1 << 30, 4)
    exb = D.DeviceExecutor(G.DeviceGraph.from_csr(gb))
    db = D.sharded_sssp(exb, 0, stats=stb)
    # the exchange fused into the relaxation over peer memory (gdx_sssp_p2p_*):
    # twice (the barrier state carries over), then the overflow rerun
    dp = D.sharded_sssp_p2p(exu, 7)
    dp2 = D.sharded_sssp_p2p(exu, 7)
    dbp = D.sharded_sssp_p2p(exb, 0)
    srcs = [0, 5, 5, 99, 4000, 17, 2048]
    bc = D.sharded_bc(exu, srcs)
    tc = D.sharded_tc(exu)
    if rank == 0:
        er, erounds = p.pr(gd, 0.85, 1e-9, 110)
        q.put((r, rounds, er, erounds, d, p.sssp(gu, 7), r2, rounds2, r3, rounds3,
               bc, p.bc(gu, srcs), tc, p.tc(gu),
               (d64, st32["width"], st64["width"], db, p.sssp(gb, 0), stb["width"], dd,
                st32["exchange"]), (dp, dp2, dbp)))
    tdist.destroy_process_group()


@pytest.mark.timeout(600)
@pytest.mark.parametrize("world", [1, 2, 3])
def test_sharded_pr_sssp_device(gdx, world):
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gpu_shard_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    r, rounds, er, erounds, d, ed, r2, rounds2, r3, rounds3, bc, ebc, tc, etc_, wide, p2p = \
        q.get(timeout=500)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert rounds == erounds == rounds2 == rounds3
    assert rel_err(r, er) < 1e-12
    assert rel_err(r2, er) < 1e-12 and rel_err(r3, er) < 1e-12
    assert np.array_equal(d, ed)
    d64, w32, w64, db, edb, wb, dd, exch = wide
    assert np.array_equal(d64, ed) and (w32, w64) == (32, 64) and np.array_equal(dd, ed)
    assert world == 1 or exch["sparse_rounds"] > 0  # delta exchange (lists < replica)
    assert np.array_equal(db, edb) and wb == 64 and edb[edb < (2**63 - 1) // 2].max() >= 2**31 - 1
    assert rel_err(bc, ebc) < 1e-9 and tc == etc_
    dp, dp2, dbp = p2p
    assert np.array_equal(dp, ed) and np.array_equal(dp2, ed) and np.array_equal(dbp, edb)


def test_tc_hub_degree_binning(gdx, port):
    """A hub whose oriented list exceeds the light-path bound (|N+| > 256) goes
    through the degree-binned k_tc_heavy; lists of very unequal length take
    the galloping intersection."""
    rng = np.random.default_rng(5)
    n = 3000
    u = np.concatenate([np.zeros(n - 1, np.int32), rng.integers(1, n, 20000).astype(np.int32)])
    v = np.concatenate([np.arange(1, n, dtype=np.int32), rng.integers(1, n, 20000).astype(np.int32)])
    for directed in (False, True):
        g = port.build_from_edges(n, u, v, None, directed)
        dg = gdx.DeviceGraph.from_csr(g)
        st = {}
        assert dg.tc(stats=st) == port.tc(g), directed
        if not directed:
            # first call: orientation (count, fill, work measure), light pairs,
            # heavy pairs; later calls reuse the cached orientation
            assert st["launches"] == 5
            st2 = {}
            assert dg.tc(stats=st2) == port.tc(g) and st2["launches"] == 2
            assert dg.tc_range(0, 1) + dg.tc_range(1, n) == port.tc(g)
            assert dg.tc_range(0, 1) == port.tc_range(g, 0, 1)


def test_memory_pool_reuse_and_trim(gdx, port):
    """Destroyed graphs' device buffers are reused by the next graph of the same
    shape (no new cudaMalloc: free memory stays flat) and gdx_pool_trim hands
    them back to the driver."""
    import ctypes as C
    torch = pytest.importorskip("torch")
    from paper_2401_02472_b200 import _lib
    u, v = port.gen_rmat_edges(1 << 14, 1 << 17, 3)
    g = port.build_from_edges(1 << 14, u, v, None, True)
    exp, it = port.pr(g, 0.85, 1e-9, 110)
    free = []
    for _ in range(4):
        dg = gdx.DeviceGraph.from_csr(g)
        got, rounds = dg.pagerank(0.85, 1e-9, 110)
        assert rounds == it and rel_err(got, exp) < 1e-12
        dg.close()
        free.append(torch.cuda.mem_get_info()[0])
    assert max(free[1:]) - min(free[1:]) < (4 << 20)  # steady state: blocks reused
    released = C.c_int64(0)
    _lib.check(_lib.load().gdx_pool_trim(C.byref(released)))
    assert released.value > 0
    assert torch.cuda.mem_get_info()[0] >= free[-1]


@pytest.mark.timeout(300)
def test_reverse_ids_past_2e9_edges(gdx):
    """RMAT-26 undirected (2.1e9 stored edges, offsets near INT32_MAX): the
    mirror ids of the undirected reverse CSR, checked on 2^24 sampled edges
    weighted towards the top of the edge range, where a midpoint (lo + hi) / 2
    would overflow int32."""
    import torch
    dg = gdx.DeviceGraph.generate("rmat", 1 << 26, 1 << 30, seed=1, directed=False)
    assert dg.m > (1 << 30) + (1 << 29)
    off, dst, rsrc, reid = dg.device_arrays(["offsets", "dests", "rev_srcs", "rev_eid"])
    dg.close()
    gen = torch.Generator(device="cuda").manual_seed(3)
    k = 1 << 24
    e = torch.cat([torch.randint(0, dg.m, (k // 2,), device="cuda", generator=gen),
                   torch.randint(dg.m - (1 << 28), dg.m, (k // 2,), device="cuda", generator=gen)])
    row = torch.searchsorted(off.long(), e, right=True) - 1
    u = dst[e].long()
    r = reid[e].long()
    assert bool(torch.all(rsrc[e] == dst[e]))
    assert bool(torch.all((off.long()[u] <= r) & (r < off.long()[u + 1])))
    assert bool(torch.all(dst[r].long() == row))
