"""CPU: pin the oracle port against the reference's golden vectors (generated
from the reference itself by tests/golden/make_golden.py) and, where the
compiled reference (oracle/_ref) is present, against live reference runs."""
from __future__ import annotations

import numpy as np
import pytest

from conftest import G, known_graph, rel_err, reverse_of, sweep_graphs

INF = (2**63 - 1) // 2


# ---- known-answer fixtures (reference tests) -----------------------------------

def test_known_sssp(port, known):
    assert list(port.sssp(known_graph(known["weighted_triangle"]), 0)) == [0, 5, 6]
    c = known["weighted_triangle_isolated"]
    got = port.sssp(known_graph(c), 0)
    assert list(got) == c["sssp0"] == c["sssp0_oracle"]
    assert got[3] == INF
    c = known["self_loops"]
    assert list(port.sssp(known_graph(c), 0)) == c["sssp0"]


def test_known_tc(port, known):
    assert port.tc(known_graph(known["k4"])) == known["k4"]["tc"] == known["k4"]["tc_oracle"] == 4
    assert port.tc(known_graph(known["self_loops"])) == known["self_loops"]["tc"]
    assert port.tc(known_graph(known["weighted_triangle"])) == 1


def test_known_bc(port, known):
    assert list(port.bc(known_graph(known["path3"]), [0, 1, 2])) == [0.0, 2.0, 0.0]
    c7 = port.bc(known_graph(known["cycle7"]), list(range(7)))
    assert np.allclose(c7, c7[0], rtol=1e-12)
    assert rel_err(c7, known["cycle7"]["bc_all"]) < 1e-12
    c = known["self_loops"]
    assert rel_err(port.bc(known_graph(c), list(range(5))), c["bc_all"]) < 1e-12


def test_known_pr(port, known):
    c = known["pr_two_cycle"]
    r, it = port.pr(known_graph(c), 0.85, 1e-9, 110)
    assert np.array_equal(r, c["pr"]) and it == c["pr_iter"]
    c = known["pr_rmat40"]
    r, it = port.pr(known_graph(c), 0.85, 1e-12, 1000)
    assert np.array_equal(r, c["pr"]), "port must be bit-identical to sequential interp::run"
    assert it == c["pr_iter"]
    assert abs(r.sum() - 1.0) < 1e-9
    # pr.sp:25: maxIter = 3 runs 4 rounds and equals oracles::pr(..., 4)
    c = known["pr_maxiter3"]
    r, it = port.pr(known_graph(c), 0.85, 0.0, 3)
    assert it == 4 == c["pr_iter"]
    assert np.array_equal(r, c["pr"]) and np.array_equal(r, c["pr_oracle4"])


def test_known_csr(port, known):
    for name, (n, u, v, w, directed) in {
        "directed_triangle": (3, [0, 0, 1], [1, 2, 2], None, True),
        "dup_min_weight": (2, [0, 0, 0], [1, 1, 1], [9, 4, 6], True),
        "self_loops": (5, [3, 0, 2, 2, 4, 1], [3, 4, 0, 2, 1, 4], [2, 7, 3, 1, 9, 4], False),
    }.items():
        g = port.build_from_edges(n, u, v, w, directed)
        exp = known[name]["graph"]
        for k in ("offsets", "dests", "weights", "rev_offsets", "rev_srcs", "rev_eid"):
            assert list(getattr(g, k)) == exp[k], (name, k)


def test_known_errors(port, known):
    from oracle import OracleError
    err = known["errors"]
    with pytest.raises(OracleError, match="InvalidEdge"):
        port.build_from_edges(2, [0], [5], None, True)
    with pytest.raises(OracleError) as e:
        port.build_from_edges(2, [0], [1], [-3], True)
    assert str(e.value) == err["negative_weight"]
    with pytest.raises(OracleError) as e:
        port.build_from_edges(2, [0], [5], None, True)
    assert str(e.value) == err["invalid_edge"]


# ---- acceptance criterion 2 sweep (acceptance_main.cpp:108-181) ------------------

def test_sweep_generators_and_csr(port, sweep):
    """makeGraph through the port == the reference's graphs, bit for bit."""
    for seed in range(1, 201):
        n = 2 + seed % 59
        m = n * (2 + seed % 3)
        u, v = port.gen_uniform_edges(n, m, seed) if seed % 2 == 0 else port.gen_rmat_edges(n, m, seed)
        und = port.with_random_weights(port.build_from_edges(n, u, v, None, False), 1, 100, seed)
        dr = port.build_from_edges(n, u, v, None, True)
        p = f"s{seed}_"
        for k in ("offsets", "dests", "weights"):
            assert np.array_equal(getattr(und, k), sweep[p + "und_" + k]), (seed, k)
            assert np.array_equal(getattr(dr, k), sweep[p + "dir_" + k]), (seed, k)


def test_sweep_algorithms(port, sweep):
    for seed in range(1, 201):
        und, dr = sweep_graphs(sweep, seed)
        p = f"s{seed}_"
        n = und.n
        assert np.array_equal(port.sssp(und, seed % n), sweep[p + "sssp"]), seed
        assert port.tc(und) == int(sweep[p + "tc"][0]) == int(sweep[p + "tc"][1]), seed
        bc = port.bc(und, list(range(n)))
        assert np.array_equal(bc, sweep[p + "bc_oracle"]), seed  # bit-identical to oracles::bc
        assert rel_err(bc, sweep[p + "bc"]) < 1e-9, seed  # interp::run tolerance (corpus.cpp:66)
        r, it = port.pr(dr, 0.85, 1e-9, 110)
        assert np.array_equal(r, sweep[p + "pr"]), seed
        assert it == int(sweep[p + "pr_iter"][0]), seed
        assert np.max(np.abs(r - sweep[p + "pr_oracle"])) <= 1e-6, seed


# ---- live reference (oracle/_ref) -------------------------------------------------

def test_ref_csr_builder_and_weights(port, ref):
    for seed, (n, m, directed) in enumerate([(1 << 12, 1 << 15, False), (1000, 7000, True),
                                             (3000, 40000, False)], start=3):
        u, v = ref.gen_rmat_edges(n, m, seed)
        rg = ref.build(n, u, v, None, directed).with_random_weights(1, 100, seed)
        pg = port.with_random_weights(port.build_from_edges(n, u, v, None, directed), 1, 100, seed)
        h = rg.host()
        for k in ("offsets", "dests", "weights", "rev_offsets", "rev_srcs", "rev_eid"):
            assert np.array_equal(getattr(h, k), getattr(pg, k)), (seed, k)


def test_ref_algorithms_medium(port, ref):
    u, v = ref.gen_rmat_edges(1 << 12, 1 << 15, 11)
    rg = ref.build(1 << 12, u, v, None, False).with_random_weights(1, 100, 11)
    h = rg.host()
    for s in (0, 1, 77):
        assert np.array_equal(port.sssp(h, s), rg.oracle_sssp(s))
    srcs = [0, 1, 2, 5, 77, 1000]
    assert np.array_equal(port.bc(h, srcs), rg.oracle_bc(srcs))
    cnt, ret = rg.interp_tc(parallel=True, threads=8)
    assert port.tc(h) == cnt == ret
    dg = ref.build(1 << 12, u, v, None, True)
    hd = dg.host()
    r, it = port.pr(hd, 0.85, 1e-9, 50)
    assert np.array_equal(r, dg.oracle_pr(0.85, 1e-9, it))


def test_ref_bfs_levels(port, ref):
    u, v = ref.gen_uniform_edges(40, 160, 5)
    g = ref.build(40, u, v, None, True)
    assert np.array_equal(port.bfs_levels(g.host(), 0), g.oracle_bfs(0))


# ---- counter-based generators (twin of the GPU generators) -------------------------

def test_ctr_generators_deterministic(port):
    u1, v1 = port.gen_rmat_ctr(1 << 10, 5000, 7, threads=4)
    u2, v2 = port.gen_rmat_ctr(1 << 10, 5000, 7, threads=1)
    assert np.array_equal(u1, u2) and np.array_equal(v1, v2)
    assert u1.max() < 1024 and (u1 < 512).mean() > 0.6  # RMAT skew toward low ids
    u, v = port.gen_rmat_ctr(1000, 4000, 7)  # non power of two: resampled in range
    assert u.max() < 1000 and v.max() < 1000
    u, v = port.gen_uniform_ctr(777, 10000, 3)
    assert u.max() < 777 and v.min() >= 0
    gu, gv = port.gen_grid_ctr(50, 0.55, 9)
    assert len(gu) == len(gv) and 0.45 < len(gu) / (2 * 50 * 49) < 0.65
    assert np.all((gv - gu == 1) | (gv - gu == 50))


def test_port_bc_no_overflow_on_grid(port):
    """on a 600x600 full grid the reference's double sigma
    overflows; the extended-exponent port stays finite and symmetric."""
    side = 600
    gu, gv = port.gen_grid_ctr(side, 1.1, 1)  # keep everything
    g = port.build_from_edges(side * side, gu, gv, None, False)
    bc = port.bc(g, [0])
    assert np.isfinite(bc).all()
    assert bc.max() > 0
