"""Robustness of the C ABI on the GPU: concurrent handles on distinct streams,
cached plans invalidated by graph mutation, input validation, memory sizing.
"""
from __future__ import annotations

import threading

import numpy as np
import pytest

from conftest import G, rel_err

pytestmark = pytest.mark.gpu


def _rmat(port, scale, seed, directed, weights=None):
    n = 1 << scale
    u, v = port.gen_rmat_edges(n, 16 * n, seed)
    g = port.build_from_edges(n, u, v, None, directed)
    if weights:
        g = port.with_random_weights(g, weights[0], weights[1], seed)
    return g


def test_concurrent_handles_on_two_streams(gdx, port):
    """Distinct handles run concurrently on their own streams from two host
    threads (gdx.h threading contract); pool releases are stream-ordered, so
    neither stalls nor corrupts the other."""
    import torch
    a = _rmat(port, 13, 3, False, (1, 100))
    b = _rmat(port, 12, 4, True)
    ea = port.sssp(a, 0)
    eb, eit = port.pr(b, 0.85, 1e-9, 110)
    errors = []

    def work_sssp():
        try:
            s = torch.cuda.Stream()
            for _ in range(6):
                g = gdx.DeviceGraph.from_csr(a)
                g.set_stream(s.cuda_stream)
                assert np.array_equal(g.sssp(0), ea)
                assert g.tc() == port.tc(a)
                g.close()
        except Exception as e:  # noqa: BLE001
            errors.append(e)

    def work_pr():
        try:
            s = torch.cuda.Stream()
            for _ in range(6):
                g = gdx.DeviceGraph.from_csr(b)
                g.set_stream(s.cuda_stream)
                r, it = g.pagerank(0.85, 1e-9, 110)
                assert it == eit and rel_err(r, eb) < 1e-9
                g.close()
        except Exception as e:  # noqa: BLE001
            errors.append(e)

    ts = [threading.Thread(target=work_sssp), threading.Thread(target=work_pr)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors


def test_sssp_after_set_hash_weights(gdx, port):
    """The cached SSSP round-loop graph is keyed on the CSR arrays: switching
    the weights on a handle after a call must not replay the old loop."""
    g0 = _rmat(port, 12, 5, False)  # max degree > 64: CUDA-graph mode
    dg = gdx.DeviceGraph.from_csr(g0)
    d_unit = dg.sssp(0)
    assert np.array_equal(d_unit, port.sssp(g0, 0))
    dg.set_hash_weights(1, 100, 7)
    h = dg.download()
    hw = G(h.n, h.m, False, h.offsets, h.dests, h.weights)
    d_w = dg.sssp(0)
    assert np.array_equal(d_w, port.sssp(hw, 0))
    assert not np.array_equal(d_w, d_unit)


def test_sssp_reweighted_in_place(gdx, port, monkeypatch):
    """Reweighting a handle in place (same weight buffer) with a larger maximum
    weight must not replay a round loop whose overflow test assumed the old
    maximum: the cached loop is keyed on it (16-bit distances forced, so the
    second weighting overflows them and the call reruns wider)."""
    monkeypatch.setenv("GDX_SSSP_NARROW", "1")
    monkeypatch.setenv("GDX_SSSP_MODE", "graph")
    gu, gv = port.gen_grid_ctr(100, 2.0, 1)
    g = port.build_from_edges(100 * 100, gu, gv, None, False)
    dg = gdx.DeviceGraph.from_csr(g)
    for lo, hi in ((1, 10), (300, 600), (1, 10)):
        dg.set_random_weights(lo, hi, 3)
        h = dg.download()
        hw = G(h.n, h.m, False, h.offsets, h.dests, h.weights)
        exp = port.sssp(hw, 0)
        assert np.array_equal(dg.sssp(0), exp), (lo, hi)


def test_undirected_view_must_be_symmetric(gdx):
    """An undirected view with a missing mirror edge is rejected (the handle
    reads the forward arrays as the reverse CSR and TC sizes from them)."""
    # upper triangle of K4 only, claimed undirected
    off = np.array([0, 3, 5, 6, 6], np.int32)
    dst = np.array([1, 2, 3, 2, 3, 3], np.int32)
    with pytest.raises(gdx.GraphdslError, match="not stored symmetrically"):
        gdx.DeviceGraph.from_csr(G(4, 6, False, off, dst))
    # the symmetric K4 is accepted
    off = np.array([0, 3, 6, 9, 12], np.int32)
    dst = np.array([1, 2, 3, 0, 2, 3, 0, 1, 3, 0, 1, 2], np.int32)
    assert gdx.DeviceGraph.from_csr(G(4, 12, False, off, dst)).tc() == 4


def test_pagerank_huge_max_iter_is_cheap(gdx, port):
    """maxIter does not size device memory (the vote flags are a ring):
    INT32_MAX - 1 runs like 100 when the ranks settle early."""
    b = _rmat(port, 12, 6, True)
    dg = gdx.DeviceGraph.from_csr(b)
    r1, it1 = dg.pagerank(0.85, 1e-6, 100)
    r2, it2 = dg.pagerank(0.85, 1e-6, 2**31 - 2)
    assert it1 == it2 and np.array_equal(r1, r2)
    # more rounds than the ring holds (threshold 0 never settles: maxIter+1 rounds)
    r3, it3 = dg.pagerank(0.85, 0.0, 700)
    e3, ie3 = port.pr(b, 0.85, 0.0, 700)
    assert it3 == ie3 == 701 and rel_err(r3, e3) < 1e-9


def test_tc_plan_cached_and_repeatable(gdx, port):
    """The oriented CSR is built by the first call and reused: repeated calls
    give the same count and report the SURVEY 8(d) bytes."""
    a = _rmat(port, 13, 8, False)
    dg = gdx.DeviceGraph.from_csr(a)
    st1, st2 = {}, {}
    c1 = dg.tc(stats=st1)
    c2 = dg.tc(stats=st2)
    assert c1 == c2 == port.tc(a)
    assert st1["algorithmic_bytes"] == st2["algorithmic_bytes"] > 0
    assert st2["launches"] < st1["launches"]


def test_pagerank_run_to_run_identical(gdx, port):
    """No floating-point atomics on the PR path: rows crossing warp chunks and
    the dangling mass are summed in a fixed order, so repeated calls (and a
    fresh handle) give bit-identical ranks."""
    b = _rmat(port, 17, 9, True)
    dg = gdx.DeviceGraph.from_csr(b)
    r1, it1 = dg.pagerank(0.85, 1e-9, 110)
    r2, it2 = dg.pagerank(0.85, 1e-9, 110)
    r3, it3 = gdx.DeviceGraph.from_csr(b).pagerank(0.85, 1e-9, 110)
    assert it1 == it2 == it3
    assert np.array_equal(r1, r2) and np.array_equal(r1, r3)
    e, ie = port.pr(b, 0.85, 1e-9, 110)
    assert ie == it1 and rel_err(r1, e) < 1e-9
