"""The in-process multi-GPU C ABI (gdx_context / gdx_*_multi, multi.cu) against
the oracle.  One B200 is available: a context of [0] exercises the NCCL
communicator path (ncclCommInitAll over one device), and contexts listing
device 0 two or three times run the full partitioned protocol -- peer
atomicMin into the owners' replicas with device-side barriers (SSSP), contrib
and partials written into every partition's buffers (PR), range counts (TC),
source blocks with a peer-memory sum (BC) -- on one GPU.
"""
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


@pytest.fixture(scope="module")
def graphs(port):
    und = _rmat(port, 13, 21, False, (1, 100))
    dr = _rmat(port, 13, 22, True)
    return und, dr


@pytest.mark.parametrize("devices", [[0], [0, 0], [0, 0, 0]])
def test_multi_matches_oracle(gdx, port, graphs, devices):
    und, dr = graphs
    ctx = gdx.Context(devices)
    info = ctx.info()
    assert info["devices"] == len(devices) and info["peer_access"]
    assert info["nccl_comms"] == (1 if devices == [0] else 0)
    mu = gdx.MultiGraph(ctx, und)
    md = gdx.MultiGraph(ctx, dr)
    for src in (0, 17, und.n - 1):
        assert np.array_equal(mu.sssp(src), port.sssp(und, src)), src
    st = {}
    mu.sssp(0, stats=st)
    assert st["rounds"] > 0 and st["algorithmic_bytes"] > 0
    assert mu.tc() == port.tc(und)
    srcs = [0, 3, 5, 8, 13, 21, 34]
    assert rel_err(mu.bc(srcs), port.bc(und, srcs)) < 1e-9
    r, it = md.pagerank(0.85, 1e-9, 110)
    re, ie = port.pr(dr, 0.85, 1e-9, 110)
    assert it == ie and rel_err(r, re) < 1e-12
    # repeated calls reuse the plans, barriers and instantiated loops
    r2, it2 = md.pagerank(0.85, 1e-9, 110)
    assert it2 == it and np.array_equal(r, r2)
    assert np.array_equal(mu.sssp(0), port.sssp(und, 0))
    mu.close()
    md.close()
    ctx.close()


def test_multi_sssp_overflow_rerun(gdx, port):
    """32-bit distances that would overflow rerun the partitioned rounds with
    64-bit distances on every device."""
    n = 300
    u = np.arange(n - 1, dtype=np.int32)
    v = u + 1
    w = np.full(n - 1, 1 << 27, np.int32)  # the path's far end is ~2^35 away
    g = port.build_from_edges(n, u, v, w, False)
    ctx = gdx.Context([0, 0])
    mg = gdx.MultiGraph(ctx, g)
    assert np.array_equal(mg.sssp(0), port.sssp(g, 0))


def test_multi_errors(gdx, port, graphs):
    und, dr = graphs
    with pytest.raises(gdx.GraphdslError, match="out of range"):
        gdx.Context([0, 99])
    ctx = gdx.Context([0, 0])
    mg = gdx.MultiGraph(ctx, und)
    with pytest.raises(gdx.GraphdslError) as e:
        mg.sssp(und.n)
    assert e.value.kind == "RuntimeError"
    two = gdx.MultiGraph(ctx, port.build_from_edges(2, [0, 1], [1, 0], None, True))
    with pytest.raises(gdx.GraphdslError) as e:
        two.pagerank(0.85, -1.0, 1000)
    assert e.value.kind == "NonTermination"
    _, it = two.pagerank(0.85, -1.0, 50)
    assert it == 51


@pytest.mark.parametrize("devices", [[0], [0, 0, 0]])
def test_multi_sssp_narrow_split(gdx, port, graphs, devices, monkeypatch):
    """The partitioned rounds with gdx_sssp's large-graph choices forced on a
    small graph: 16-bit distances first and the small vertices' second queue
    (GDX_SSSP_NARROW=1, GDX_SSSP_SPLIT=1).  A path whose far end lies beyond
    2^16 overflows the 16-bit attempt and reruns at 32 bits on every
    partition."""
    monkeypatch.setenv("GDX_SSSP_NARROW", "1")
    monkeypatch.setenv("GDX_SSSP_SPLIT", "1")
    und, _ = graphs
    ctx = gdx.Context(devices)
    mu = gdx.MultiGraph(ctx, und)
    for src in (0, 17, und.n - 1):
        assert np.array_equal(mu.sssp(src), port.sssp(und, src)), src
    n = 3000
    u = np.arange(n - 1, dtype=np.int32)
    w = np.full(n - 1, 100, np.int32)  # far end 299,900 away
    g = port.build_from_edges(n, u, u + 1, w, False)
    mg = gdx.MultiGraph(ctx, g)
    ref = port.sssp(g, 0)
    assert ref.max() > 1 << 16
    assert np.array_equal(mg.sssp(0), ref)
    assert np.array_equal(mg.sssp(0), ref)  # the handle remembers the overflow
    mu.close()
    mg.close()
    ctx.close()
