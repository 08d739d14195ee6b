"""GPU parity at the BASELINE.json configurations themselves:
every config's full result against the oracle on the same graph.

  C1  SSSP on the reference's own RMAT-18 graph + weights: exact, and equal to
      the reference's interp::run when oracle/_ref is built
  C2  PageRank RMAT-24 (2^28 draws): same round count, ranks <= 1e-6 relative
  C3  TC uniform 2^24 / 2^27 draws: exact count
  C4  BC on the 4899^2 grid: 16 of the bench's 64 sources, <= 1e-6 relative
  C5  SSSP RMAT-26 (~2.1e9 edges): exact against Dijkstra

Minutes, not seconds: the oracle runs on the host's cores.
"""
from __future__ import annotations

import os

import numpy as np
import pytest

from conftest import rel_err

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
CORES = os.cpu_count() or 1


def test_c1_sssp_reference_graph(gdx, port):
    import paper_2401_02472_b200 as g
    u, v = g.gen_rmat_edges(1 << 18, 1 << 22, 1)
    dg = gdx.DeviceGraph.build_from_edges(1 << 18, u, v, None, directed=False)
    dg.set_random_weights(1, 100, 1)
    h = dg.download(("offsets", "dests", "weights"))
    # the product path builds exactly the oracle's (= the reference's) C1 graph
    pu, pv = port.gen_rmat_edges(1 << 18, 1 << 22, 1)
    exp = port.with_random_weights(port.build_from_edges(1 << 18, pu, pv, None, False), 1, 100, 1)
    assert h.m == exp.m == 7_611_081
    for k in ("offsets", "dests", "weights"):
        assert np.array_equal(getattr(h, k), getattr(exp, k)), k
    d = dg.sssp(0)
    assert np.array_equal(d, port.sssp(exp, 0))
    from oracle import Ref, ref_available
    if ref_available():
        rg = Ref().build_from_host(exp)
        di, mod, fin = rg.interp_sssp(0, parallel=True, threads=CORES)
        assert np.array_equal(d, di) and not mod.any() and fin


def test_c2_pagerank(gdx, port):
    dg = gdx.DeviceGraph.generate("rmat", 1 << 24, 1 << 28, seed=1, directed=True)
    r, it = dg.pagerank(0.85, 1e-6, 100)
    h = dg.download(("offsets", "rev_offsets", "rev_srcs"))
    dg.close()
    re, ie = port.pr(h, 0.85, 1e-6, 100, threads=CORES)
    assert it == ie
    assert rel_err(r, re) <= 1e-6
    assert abs(r.sum() - 1.0) < 1e-9


def test_c3_triangle_count(gdx, port):
    dg = gdx.DeviceGraph.generate("uniform", 1 << 24, 1 << 27, seed=1, directed=False)
    c = dg.tc()
    assert dg.tc() == c  # second call reuses the cached orientation
    h = dg.download(("offsets", "dests"))
    dg.close()
    assert c == port.tc(h, threads=CORES)


def test_c4_bc_sources(gdx, port):
    dg = gdx.DeviceGraph.generate("grid", 4899, seed=1, keep=0.55, directed=False)
    h = dg.download(("offsets", "dests"))
    cand = np.flatnonzero(np.diff(h.offsets) > 0)
    sources = sorted(np.random.default_rng(1).choice(cand, size=64, replace=False).tolist())
    sub = sources[::4]  # 16 of the bench's 64 sources
    b = dg.bc(sub)
    dg.close()
    e = port.bc(h, sub, threads=CORES)
    assert np.isfinite(b).all()
    assert rel_err(b, e) <= 1e-6


def test_c5_sssp_dijkstra(gdx, port):
    dg = gdx.DeviceGraph.generate("rmat", 1 << 26, 1 << 30, seed=1, directed=False,
                                  weights=(1, 100))
    assert dg.m > 2_000_000_000
    d = dg.sssp(0)
    h = dg.download(("offsets", "dests", "weights"))
    dg.close()
    assert np.array_equal(d, port.sssp(h, 0))
