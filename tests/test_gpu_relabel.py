"""The degree-ordered renumbering cached on a handle (csrc/relabel.cu) against
the oracle: PageRank and SSSP run on the renumbered graph and map their
results back.  It is on by default only for skewed graphs of >= 2^22 vertices
(the C2 / C5 bench graphs, whose parity bench.py checks every run); here
GDX_RELABEL=1 forces it on graphs the oracle finishes in seconds.

Bars as in test_gpu_parity.py: SSSP bit-exact, PageRank the same round count
and within 1e-9 relative (only the summation order differs)."""
from __future__ import annotations

import numpy as np
import pytest

from conftest import rel_err

pytestmark = pytest.mark.gpu


def _rmat(port, scale, seed, directed, weights=None):
    n = 1 << scale
    u, v = port.gen_rmat_edges(n, 16 * n, seed)
    g = port.build_from_edges(n, u, v, None, directed)
    if weights:
        g = port.with_random_weights(g, weights[0], weights[1], seed)
    return g


@pytest.fixture
def relabel_on(monkeypatch):
    monkeypatch.setenv("GDX_RELABEL", "1")


@pytest.mark.parametrize("directed", [True, False])
def test_pagerank_relabelled(gdx, port, relabel_on, directed):
    import torch
    g = _rmat(port, 14, 3, directed)
    dg = gdx.DeviceGraph.from_csr(g)
    st = {}
    r, it = dg.pagerank(0.85, 1e-9, 110, stats=st)
    re, ie = port.pr(g, 0.85, 1e-9, 110)
    assert it == ie and rel_err(r, re) < 1e-9
    # repeated calls reuse the renumbered graph and its plan: identical results
    r2, it2 = dg.pagerank(0.85, 1e-9, 110)
    assert it2 == it and np.array_equal(r, r2)
    # device output
    out = torch.empty(g.n, dtype=torch.float64, device="cuda")
    dg.pagerank(0.85, 1e-9, 110, out=out)
    assert np.array_equal(out.cpu().numpy(), r)
    dg.close()


def test_pagerank_relabel_profiled(gdx, port, relabel_on):
    """The renumbered graph's kernels appear in the owner's profile."""
    g = _rmat(port, 12, 4, True)
    dg = gdx.DeviceGraph.from_csr(g)
    dg.profile(True)
    dg.pagerank(0.85, 1e-9, 110)
    prof = dg.profile_read()
    assert "relabel" in prof and "pr_edges" in prof and "pr_unpermute" in prof
    dg.profile_reset()
    dg.pagerank(0.85, 1e-9, 110)
    prof = dg.profile_read()
    assert "relabel" not in prof and prof["pr_edges"][1] > 0
    dg.close()


@pytest.mark.parametrize("narrow", ["0", "1"])
def test_sssp_relabelled(gdx, port, relabel_on, monkeypatch, narrow):
    import torch
    monkeypatch.setenv("GDX_SSSP_NARROW", narrow)
    monkeypatch.setenv("GDX_SSSP_SPLIT", narrow)
    g = _rmat(port, 14, 5, False, (1, 100))
    dg = gdx.DeviceGraph.from_csr(g)
    for src in (0, 17, g.n - 1):
        assert np.array_equal(dg.sssp(src), port.sssp(g, src)), src
    out = torch.empty(g.n, dtype=torch.int64, device="cuda")
    dg.sssp(5, out=out)
    assert np.array_equal(out.cpu().numpy(), port.sssp(g, 5))
    # new weights invalidate the renumbered copy (it holds the old ones)
    dg.set_random_weights(1, 1000, 9)
    g2 = port.with_random_weights(g, 1, 1000, 9)
    assert np.array_equal(dg.sssp(0), port.sssp(g2, 0))
    dg.close()


def test_sssp_relabelled_directed_unweighted(gdx, port, relabel_on):
    g = _rmat(port, 13, 6, True)
    dg = gdx.DeviceGraph.from_csr(g)
    for src in (0, 1, 100):
        assert np.array_equal(dg.sssp(src), port.sssp(g, src)), src
    dg.close()


def test_relabel_off_matches(gdx, port, monkeypatch):
    """GDX_RELABEL=0 and =1 give the same distances and round counts."""
    g = _rmat(port, 13, 7, False, (1, 50))
    res = {}
    for flag in ("0", "1"):
        monkeypatch.setenv("GDX_RELABEL", flag)
        dg = gdx.DeviceGraph.from_csr(g)
        res[flag] = (dg.sssp(3), dg.pagerank(0.85, 1e-9, 110))
        dg.close()
    assert np.array_equal(res["0"][0], res["1"][0])
    assert res["0"][1][1] == res["1"][1][1] and rel_err(res["0"][1][0], res["1"][1][0]) < 1e-12


def _relabel_shard_worker(rank, world, port, q):
    import os
    import sys
    from conftest import ROOT
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK="0", GDX_RELABEL="1")
    import torch.distributed as tdist
    import paper_2401_02472_b200 as G
    from paper_2401_02472_b200 import distributed as D
    from oracle import Port
    D.init_from_env("gloo")  # the ranks share cuda:0 (see test_gpu_parity.py)
    p = Port()
    n = 1 << 12
    u, v = p.gen_rmat_edges(n, 16 * n, 31)
    gd = p.build_from_edges(n, u, v, None, True)
    gu = p.with_random_weights(p.build_from_edges(n, u, v, None, False), 1, 100, 31)
    exd = D.DeviceExecutor(G.DeviceGraph.from_csr(gd))
    r, rounds = D.sharded_pr_p2p(exd, 0.85, 1e-9, 110)
    r2, rounds2 = D.sharded_pr_p2p(exd, 0.85, 1e-9, 110)
    single, srounds = exd.g.pagerank(0.85, 1e-9, 110)
    exu = D.DeviceExecutor(G.DeviceGraph.from_csr(gu))
    d = D.sharded_sssp_p2p(exu, 7)
    d2 = D.sharded_sssp_p2p(exu, 9)
    if rank == 0:
        er, erounds = p.pr(gd, 0.85, 1e-9, 110)
        q.put((r, rounds, r2, rounds2, single, srounds, er, erounds, d, p.sssp(gu, 7), d2,
               p.sssp(gu, 9)))
    tdist.destroy_process_group()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("world", [1, 2])
def test_sharded_on_renumbered_graph(gdx, world):
    """The peer-memory PR / SSSP partitions run on the renumbered graph the
    single-GPU calls use (distributed._renumbered) and map results back."""
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_relabel_shard_worker, args=(r, world, port, q))
             for r in range(world)]
    for pr in procs:
        pr.start()
    r, rounds, r2, rounds2, single, srounds, er, erounds, d, ed, d2, ed2 = q.get(timeout=250)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert rounds == rounds2 == srounds == erounds
    assert rel_err(r, er) < 1e-9 and rel_err(single, er) < 1e-9 and np.array_equal(r, r2)
    assert np.array_equal(d, ed) and np.array_equal(d2, ed2)


@pytest.mark.parametrize("devices", [[0], [0, 0]])
def test_multi_on_renumbered_graph(gdx, port, relabel_on, devices):
    """The in-process gdx_sssp_multi / gdx_pagerank_multi partition the
    replicas' renumbering and map the results back."""
    und = _rmat(port, 13, 8, False, (1, 100))
    dr = _rmat(port, 13, 9, True)
    ctx = gdx.Context(devices)
    mu = gdx.MultiGraph(ctx, und)
    md = gdx.MultiGraph(ctx, dr)
    for src in (0, 17, und.n - 1):
        assert np.array_equal(mu.sssp(src), port.sssp(und, src)), src
    r, it = md.pagerank(0.85, 1e-9, 110)
    re, ie = port.pr(dr, 0.85, 1e-9, 110)
    assert it == ie and rel_err(r, re) < 1e-9
    r2, it2 = md.pagerank(0.85, 1e-9, 110)
    assert it2 == it and np.array_equal(r, r2)
    mu.close()
    md.close()
    ctx.close()


def test_auto_policy_at_size(gdx, monkeypatch):
    """Default policy on a skewed graph of 2^22 vertices: the first call runs
    on the caller's numbering, the second builds the renumbering and runs on
    it (the profile shows the build), later calls reuse it.  SSSP distances
    identical across all calls, PageRank within 1e-12 with the same rounds
    (bit-identical from the second call on)."""
    import torch
    monkeypatch.delenv("GDX_RELABEL", raising=False)
    n = 1 << 22
    du = gdx.DeviceGraph.generate("rmat", n, 16 * n, seed=3, directed=False, weights=(1, 100))
    out = [torch.empty(n, dtype=torch.int64, device="cuda") for _ in range(3)]
    du.profile(True)
    du.sssp(0, out=out[0])
    assert "relabel" not in du.profile_read()
    du.sssp(0, out=out[1])
    assert "relabel" in du.profile_read()
    du.sssp(0, out=out[2])
    assert torch.equal(out[0], out[1]) and torch.equal(out[1], out[2])
    du.close()
    dd = gdx.DeviceGraph.generate("rmat", n, 16 * n, seed=4, directed=True)
    r = [dd.pagerank(0.85, 1e-6, 100) for _ in range(3)]
    assert r[0][1] == r[1][1] == r[2][1]
    assert rel_err(r[0][0], r[1][0]) < 1e-12 and np.array_equal(r[1][0], r[2][0])
    dd.close()


def test_renumbering_out_of_memory_falls_back(gdx, port, relabel_on, monkeypatch):
    """A renumbering build that runs out of device memory leaves the call on
    the caller's numbering (same results) and the handle stops trying."""
    monkeypatch.setenv("GDX_RELABEL_TEST_OOM", "1")
    g = _rmat(port, 12, 10, False, (1, 100))
    dg = gdx.DeviceGraph.from_csr(g)
    dg.profile(True)
    assert np.array_equal(dg.sssp(0), port.sssp(g, 0))
    r, it = dg.pagerank(0.85, 1e-9, 110)
    re, ie = port.pr(g, 0.85, 1e-9, 110)
    assert it == ie and rel_err(r, re) < 1e-9
    assert dg.renumbered("sssp") is None and "relabel" not in dg.profile_read()
    dg.close()
