"""CPU, world_size 2 over gloo: the multi-GPU sharding and collective logic of
paper_2401_02472_b200.distributed, with the per-rank compute supplied by the
oracle port (the GPU executor is the only part not exercised here)."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
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

    def rev_offsets(self):
        return self.g.rev_offsets

    def num_nodes(self):
        return self.g.n

    # --- PR shard: numpy restatement of gdx_pr_shard_* (pr.sp:17-30 per row) ---
    def pr_setup(self, v0, v1):
        self.v0, self.v1 = v0, v1

    def pr_init(self, contrib_slice, partials):
        n, v0, v1 = self.g.n, self.v0, self.v1
        r0 = 1.0 / n
        od = np.diff(self.g.offsets)[v0:v1]
        contrib_slice[:v1 - v0] = torch.from_numpy(np.where(od > 0, r0 / np.maximum(od, 1), 0.0))
        partials[0] = r0 * float((od == 0).sum())
        partials[1] = 0.0
        self.rank = np.full(v1 - v0, r0)

    def pr_round(self, rnd, damping, threshold, max_iter, dangling_in, contrib, contrib_slice,
                 partials):
        n, v0, v1 = self.g.n, self.v0, self.v1
        c = contrib.numpy()
        roff, src = self.g.rev_offsets, self.g.rev_srcs
        sums = np.zeros(v1 - v0)
        for i, v in enumerate(range(v0, v1)):
            sums[i] = c[src[roff[v]:roff[v + 1]]].sum()
        new = (1.0 - damping) / n + damping * (float(dangling_in[0]) / n + sums)
        unsettled = bool(np.any(np.abs(new - self.rank) >= threshold)) and rnd < max_iter
        od = np.diff(self.g.offsets)[v0:v1]
        contrib_slice[:v1 - v0] = torch.from_numpy(np.where(od > 0, new / np.maximum(od, 1), 0.0))
        partials[0] = float(new[od == 0].sum())
        partials[1] = 1.0 if unsettled else 0.0
        self.rank = new

    def pr_rank(self, rounds, rank_slice):
        rank_slice[:self.v1 - self.v0] = torch.from_numpy(self.rank)

    # --- SSSP shard: numpy restatement of gdx_sssp_shard_* ---
    def sssp_setup(self, v0, v1):
        self.s0, self.s1 = v0, v1
        self.ovf = 0

    def sssp_frontier(self, dist, prev):
        d, p = dist.numpy(), prev.numpy()
        own = np.arange(self.s0, self.s1)
        self.front = own[d[own] < p[own]]
        p[self.front] = d[self.front]
        return len(self.front)

    def sssp_relax(self, dist):
        d = dist.numpy()
        off, dst = self.g.offsets, self.g.dests
        w = self.g.weights if self.g.weights is not None else np.ones(self.g.m, np.int32)
        for v in self.front:
            e = slice(off[v], off[v + 1])
            np.minimum.at(d, dst[e], d[v] + w[e].astype(np.int64))

    # int32 replicas (gdx_sssp_shard_*32): INF = INT32_MAX, a relaxation that
    # would reach it raises the overflow flag reported by the next frontier call
    def sssp_frontier32(self, dist, prev):
        c = self.sssp_frontier(dist, prev)
        o, self.ovf = self.ovf, 0
        return c, o

    def sssp_relax32_delta(self, dist, ids, vals):
        """gdx_sssp_shard_relax32_delta: the relaxation plus the list of the
        vertices whose replica distance it lowered (once each) and their values."""
        before = dist.numpy().copy()
        self.sssp_relax32(dist)
        d = dist.numpy()
        ch = np.flatnonzero(d < before).astype(np.int32)
        ids[:len(ch)] = torch.from_numpy(ch)
        vals[:len(ch)] = torch.from_numpy(d[ch])
        return len(ch)

    def sssp_apply32(self, dist, ids, vals, count):
        d, i, v = dist.numpy(), ids.numpy()[:count], vals.numpy()[:count]
        np.minimum.at(d, i[i >= 0], v[i >= 0])

    def sssp_relax32(self, dist):
        d = dist.numpy()
        off, dst = self.g.offsets, self.g.dests
        w = self.g.weights if self.g.weights is not None else np.ones(self.g.m, np.int32)
        for v in self.front:
            e = slice(off[v], off[v + 1])
            c = int(d[v]) + w[e].astype(np.int64)
            ok = c < D.INF32
            self.ovf |= int(not ok.all())
            np.minimum.at(d, dst[e][ok], c[ok].astype(np.int32))


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


def _worker_pr_sssp(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    import torch.distributed as dist
    from oracle import Port
    D.init_from_env("gloo")
    p = Port()
    n = 1 << 10
    u, v = p.gen_rmat_edges(n, 8 * n, 9)
    gd = p.build_from_edges(n, u, v, None, True)
    rank_v, rounds = D.sharded_pr(OracleExecutor(gd), 0.85, 1e-9, 110)
    gu = p.with_random_weights(p.build_from_edges(n, u, v, None, False), 1, 100, 9)
    st0, st5, st64, stbig = {}, {}, {}, {}
    d0 = D.sharded_sssp(OracleExecutor(gu), 0, stats=st0)
    d5 = D.sharded_sssp(OracleExecutor(gu), 5, stats=st5)
    d0w = D.sharded_sssp(OracleExecutor(gu), 0, width=64, stats=st64)
    std = {}
    d0d = D.sharded_sssp(OracleExecutor(gu), 0, exchange="dense", stats=std)
    # weights near 2^30: int32 replicas overflow, the call reruns over int64
    gb = p.with_random_weights(p.build_from_edges(n, u, v, None, False), 1 << 29, 1 << 30, 4)
    db = D.sharded_sssp(OracleExecutor(gb), 0, stats=stbig)
    if rank == 0:
        exp_r, exp_rounds = p.pr(gd, 0.85, 1e-9, 110)
        e0 = p.sssp(gu, 0)
        assert np.array_equal(d0w, e0) and st64["width"] == 64
        assert np.array_equal(d0d, e0) and std["exchange"]["sparse_rounds"] == 0
        assert st0["exchange"]["sparse_rounds"] > 0  # the delta exchange ran
        assert st0["width"] == 32 and st5["width"] == 32
        eb = p.sssp(gb, 0)
        assert np.array_equal(db, eb) and stbig["width"] == 64
        assert eb[eb < D.INF64].max() >= D.INF32  # the case really overflows int32
        q.put((rank_v, rounds, exp_r, exp_rounds, d0, e0, d5, p.sssp(gu, 5)))
    dist.destroy_process_group()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("world", [2, 3])
def test_sharded_pr_sssp_gloo(world):
    """Vertex-range PR (all-gather of contrib slices + all-reduce of the
    partials) and SSSP (MIN all-reduce of the dist replicas) against the
    single-process oracle: same PR rounds, PR within 1e-12, SSSP bit-exact."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker_pr_sssp, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    r, rounds, er, erounds, d0, e0, d5, e5 = q.get(timeout=240)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert rounds == erounds
    assert float(np.max(np.abs(r - er) / np.abs(er))) < 1e-12
    assert np.array_equal(d0, e0) and np.array_equal(d5, e5)


def test_pr_ranges_balance_in_edges():
    roff = np.array([0, 50, 50, 51, 52, 100], np.int64)
    r = D.pr_ranges(roff, 2)
    assert r[0][0] == 0 and r[-1][1] == 5 and r[0][1] == r[1][0]


def test_balanced_ranges_device_matches_numpy():
    rng = np.random.default_rng(3)
    deg = rng.integers(0, 50, size=5000)
    off = np.concatenate([[0], np.cumsum(deg)]).astype(np.int32)
    for parts in (1, 2, 3, 8):
        assert D.balanced_ranges_device(torch.from_numpy(off), parts) == D.vertex_ranges(off, parts)
