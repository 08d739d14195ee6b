"""CPU, world_size 2 over gloo: the multi-GPU sharding and collective logic of
paper_2401_02472_b200.distributed, with the per-rank compute supplied by the
oracle port (the GPU executor is the only part not exercised here)."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import ROOT

from paper_2401_02472_b200 import distributed as D


def free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_balanced_ranges_cover_and_balance():
    w = np.array([1, 1, 1, 10, 1, 1, 1, 1, 1, 1], float)
    r = D.balanced_ranges(w, 3)
    assert r[0][0] == 0 and r[-1][1] == len(w)
    assert all(a[1] == b[0] for a, b in zip(r, r[1:]))
    assert D.balanced_ranges(np.zeros(0), 4) == [(0, 0)] * 4
    rr = D.balanced_ranges(np.ones(5), 8)  # more parts than items: empty ranges ok
    assert rr[0][0] == 0 and rr[-1][1] == 5 and sum(b - a for a, b in rr) == 5
    off = np.array([0, 100, 101, 102, 103, 203], np.int64)
    w = np.diff(off) + 1.0
    r = D.vertex_ranges(off, 2)
    loads = [w[a:b].sum() for a, b in r]
    assert max(loads) <= w.sum() / 2 + w.max()
    assert r == [(0, 3), (3, 5)]


def test_source_blocks_preserve_order():
    b = D.source_blocks([5, 1, 9, 9, 2, 7, 3], 3)
    assert b == [[5, 1, 9], [9, 2], [7, 3]]
    assert sum(b, []) == [5, 1, 9, 9, 2, 7, 3]
    assert D.source_blocks([1], 4) == [[1], [], [], []]


class OracleExecutor:
    """Test double for DeviceExecutor backed by the CPU port."""

    def __init__(self, g):
        from oracle import Port
        self.p = Port()
        self.g = g

    def tc_range(self, v0, v1):
        return self.p.tc_range(self.g, v0, v1, threads=2)

    def bc(self, sources):
        return self.p.bc(self.g, sources, threads=2)

    def offsets(self):
        return self.g.offsets

    def num_nodes(self):
        return self.g.n


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    import torch.distributed as dist
    from oracle import Port
    D.init_from_env("gloo")
    p = Port()
    n = 1 << 11
    u, v = p.gen_rmat_edges(n, 16 * n, 5)
    g = p.build_from_edges(n, u, v, None, False)
    ex = OracleExecutor(g)
    tc = D.sharded_tc(ex)
    srcs = [0, 3, 3, 17, 100, 2047, 512]
    bc = D.sharded_bc(ex, srcs)
    if rank == 0:
        q.put((tc, p.tc(g), bc, p.bc(g, srcs)))
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_sharded_tc_bc_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    tc, tc_exp, bc, bc_exp = q.get(timeout=240)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert tc == tc_exp
    scale = np.maximum(np.maximum(np.abs(bc), np.abs(bc_exp)), 1e-12)
    assert float(np.max(np.abs(bc - bc_exp) / scale)) < 1e-12
