"""CPU: libgdx's host-side copies of the reference's sequential streams
(genUniformEdges / genRmatEdges / withRandomWeights, refstream.cu) reproduce
the reference's golden graphs and weights exactly.  Host code only: no GPU."""
from __future__ import annotations

import numpy as np
import pytest


def _golden_edges(gdx, seed, max_nodes=60):
    """acceptance_main.cpp:62-67 through the product's generators."""
    n = 2 + seed % (max_nodes - 1)
    m = n * (2 + seed % 3)
    if seed % 2 == 0:
        return n, gdx.gen_uniform_edges(n, m, seed)
    return n, gdx.gen_rmat_edges(n, m, seed)


def test_streams_reproduce_golden_sweep(port, sweep):
    import paper_2401_02472_b200 as gdx
    for seed in range(1, 201):
        p = f"s{seed}_"
        n, (u, v) = _golden_edges(gdx, seed)
        und = port.build_from_edges(n, u, v, None, False)
        dr = port.build_from_edges(n, u, v, None, True)
        assert np.array_equal(und.offsets, sweep[p + "und_offsets"]), seed
        assert np.array_equal(und.dests, sweep[p + "und_dests"]), seed
        assert np.array_equal(dr.dests, sweep[p + "dir_dests"]), seed
        w = gdx.random_weights(und, 1, 100, seed)
        assert np.array_equal(w, sweep[p + "und_weights"]), seed


def test_streams_match_port_at_scale(port):
    import paper_2401_02472_b200 as gdx
    n = 1 << 14
    u, v = gdx.gen_rmat_edges(n, 16 * n, 3)
    pu, pv = port.gen_rmat_edges(n, 16 * n, 3)
    assert np.array_equal(u, pu) and np.array_equal(v, pv)
    u2, v2 = gdx.gen_uniform_edges(n, 8 * n, 4)
    qu, qv = port.gen_uniform_edges(n, 8 * n, 4)
    assert np.array_equal(u2, qu) and np.array_equal(v2, qv)
    for directed in (False, True):
        g = port.build_from_edges(n, u, v, None, directed)
        assert np.array_equal(gdx.random_weights(g, 1, 100, 9),
                              port.with_random_weights(g, 1, 100, 9).weights)


def test_streams_match_reference_library(ref):
    import paper_2401_02472_b200 as gdx
    n = 1 << 12
    u, v = gdx.gen_rmat_edges(n, 16 * n, 11)
    ru, rv = ref.gen_rmat_edges(n, 16 * n, 11)
    assert np.array_equal(u, ru) and np.array_equal(v, rv)
    g = ref.build(n, u, v, None, False)
    assert np.array_equal(gdx.random_weights(g.host(), 5, 50, 2),
                          g.with_random_weights(5, 50, 2).host().weights)


def test_stream_errors_mirror_reference():
    import paper_2401_02472_b200 as gdx
    with pytest.raises(gdx.GraphdslError, match="node count must be positive"):
        gdx.gen_rmat_edges(0, 4, 1)
    with pytest.raises(gdx.GraphdslError, match="node count must be positive"):
        gdx.gen_uniform_edges(-1, 4, 1)
    with pytest.raises(gdx.GraphdslError, match="RMAT parameters must sum"):
        gdx.gen_rmat_edges(4, 4, 1, 0.0, 0.0, 0.0, 0.0)

    class G:
        n, m, directed = 2, 1, True
        offsets = np.array([0, 1, 1], np.int32)
        dests = np.array([1], np.int32)
    with pytest.raises(gdx.GraphdslError, match="weight range is empty"):
        gdx.random_weights(G, 5, 4, 1)
