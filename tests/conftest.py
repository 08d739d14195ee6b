"""Shared fixtures.  `-m gpu` tests need a B200 and the built libgdx.so;
everything else runs on the CPU (the driver runs `-m "not gpu"` here)."""
from __future__ import annotations

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 and the built libgdx.so")
    config.addinivalue_line("markers", "slow: large-graph test (seconds to minutes)")


class G:
    """Minimal CsrGraph-shaped record (numpy arrays)."""

    def __init__(self, n, m, directed, offsets, dests, weights=None, rev_offsets=None,
                 rev_srcs=None, rev_eid=None):
        self.n, self.m, self.directed = int(n), int(m), bool(directed)
        self.offsets = np.asarray(offsets, np.int32)
        self.dests = np.asarray(dests, np.int32)
        self.weights = None if weights is None else np.asarray(weights, np.int32)
        self.rev_offsets = None if rev_offsets is None else np.asarray(rev_offsets, np.int32)
        self.rev_srcs = None if rev_srcs is None else np.asarray(rev_srcs, np.int32)
        self.rev_eid = None if rev_eid is None else np.asarray(rev_eid, np.int32)


def reverse_of(g: G) -> G:
    """csr.cpp:77-94 in numpy (stable transpose)."""
    src = np.repeat(np.arange(g.n, dtype=np.int64), np.diff(g.offsets))
    order = np.lexsort((src, g.dests))
    rev_off = np.zeros(g.n + 1, np.int64)
    np.add.at(rev_off, g.dests.astype(np.int64) + 1, 1)
    g.rev_offsets = np.cumsum(rev_off).astype(np.int32)
    g.rev_srcs = src[order].astype(np.int32)
    g.rev_eid = order.astype(np.int32)
    return g


@pytest.fixture(scope="session")
def port():
    from oracle import Port
    return Port()


@pytest.fixture(scope="session")
def ref():
    from oracle import Ref, ref_available
    if not ref_available():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return Ref()


@pytest.fixture(scope="session")
def known():
    with open(os.path.join(GOLDEN, "known.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def sweep():
    return dict(np.load(os.path.join(GOLDEN, "sweep.npz")))


def known_graph(case: dict) -> G:
    g = case["graph"]
    return G(g["n"], g["m"], g["directed"], g["offsets"], g["dests"], g["weights"],
             g["rev_offsets"], g["rev_srcs"], g["rev_eid"])


def sweep_graphs(sweep: dict, seed: int):
    p = f"s{seed}_"
    n, mu, md = (int(x) for x in sweep[p + "n"])
    und = reverse_of(G(n, mu, False, sweep[p + "und_offsets"], sweep[p + "und_dests"],
                       sweep[p + "und_weights"]))
    dr = reverse_of(G(n, md, True, sweep[p + "dir_offsets"], sweep[p + "dir_dests"],
                      sweep[p + "dir_weights"]))
    return und, dr


def rel_err(a, b) -> float:
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    if a.size == 0:
        return 0.0
    scale = np.maximum(np.maximum(np.abs(a), np.abs(b)), 1e-12)
    return float(np.max(np.abs(a - b) / scale))


@pytest.fixture(scope="session")
def gdx():
    """The product package, with a GPU present (fails loudly otherwise)."""
    import paper_2401_02472_b200 as gdx_pkg
    assert gdx_pkg.device_count() >= 1, "no CUDA device visible"
    return gdx_pkg
