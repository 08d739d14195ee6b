"""Multi-GPU sharding of the corpus algorithms (one process per GPU).

SURVEY.md §8(e): each algorithm shards naturally --

* TC: the graph is replicated; middle vertices are split into contiguous ranges
  balanced by their oriented work; every rank counts its range
  (``gdx_tc_range``) and one int64 all-reduce sums the counts.  No per-round
  exchange.
* BC: the graph is replicated; the source set is split into contiguous blocks
  (source order preserved inside a block); every rank accumulates a partial
  ``bc`` and one f64 all-reduce of n sums them.  The cross-rank sum order
  differs from the reference's source order only by rounding (within 1e-6).
* PR: destination-vertex ranges balanced by in-edges; every rank computes its
  rows from the full contrib vector (``gdx_pr_shard_round``); per round one
  all-gather of the contrib slices and one all-reduce of (dangling mass,
  unsettled vote).  Same arithmetic and round count as ``gdx_pagerank``.
* SSSP: vertex ranges balanced by out-edges; every rank keeps a replica of
  dist, relaxes the out-edges of its own improved vertices
  (``gdx_sssp_shard_*``), and one element-wise MIN all-reduce merges the
  replicas per round; one SUM all-reduce of the improvement counts decides
  the fixedPoint.  Distances are unique, so the result is bit-exact.

``torch.distributed`` carries the collectives: NCCL over NVLink on the GPU box,
gloo on the CPU for the tests.  The per-rank compute is pluggable so the
sharding and collective logic can be exercised on the CPU (tests inject an
oracle-backed executor); the product executor is ``DeviceExecutor`` (libgdx.so
on this rank's GPU).
"""
from __future__ import annotations

from typing import Optional, Protocol, Sequence

import numpy as np


# ---------------------------------------------------------------------------- partitioners

def balanced_ranges(weights: np.ndarray, parts: int) -> list[tuple[int, int]]:
    """Split [0, len(weights)) into `parts` contiguous ranges of ~equal total
    weight (prefix-sum cut points; empty ranges allowed)."""
    n = len(weights)
    if parts <= 0:
        raise ValueError("parts must be positive")
    if n == 0:
        return [(0, 0)] * parts
    csum = np.concatenate([[0], np.cumsum(np.asarray(weights, dtype=np.float64))])
    total = csum[-1]
    cuts = [0]
    for p in range(1, parts):
        cuts.append(int(np.searchsorted(csum, total * p / parts, side="left")))
    cuts.append(n)
    cuts = np.maximum.accumulate(np.clip(cuts, 0, n))
    return [(int(cuts[i]), int(cuts[i + 1])) for i in range(parts)]


def tc_ranges(offsets: np.ndarray, parts: int) -> list[tuple[int, int]]:
    """Owner-vertex ranges for TC (gdx_tc_range) balanced by work ~ deg(v)^2 / 2 +
    deg(v) (each of ~deg/2 neighbours on one side intersects two ~deg/2 lists)."""
    deg = np.diff(np.asarray(offsets, dtype=np.int64)).astype(np.float64)
    return balanced_ranges(deg * deg / 2.0 + deg + 1.0, parts)


def vertex_ranges(offsets: np.ndarray, parts: int) -> list[tuple[int, int]]:
    """Vertex ranges balanced by (edges + vertices), the PR/SSSP partition."""
    deg = np.diff(np.asarray(offsets, dtype=np.int64)).astype(np.float64)
    return balanced_ranges(deg + 1.0, parts)


def source_blocks(sources: Sequence[int], parts: int) -> list[list[int]]:
    """Contiguous blocks of the source set (order preserved), sizes differ by <= 1."""
    src = list(sources)
    q, r = divmod(len(src), parts)
    out, i = [], 0
    for p in range(parts):
        k = q + (1 if p < r else 0)
        out.append(src[i:i + k])
        i += k
    return out


# ---------------------------------------------------------------------------- executors

class Executor(Protocol):
    """Per-rank compute.  Tensors are torch tensors on the collective device
    (CUDA under NCCL, CPU under gloo)."""

    def tc_range(self, v0: int, v1: int) -> int: ...

    def bc(self, sources: Sequence[int]) -> np.ndarray: ...

    def offsets(self) -> np.ndarray: ...

    def rev_offsets(self) -> np.ndarray: ...

    def num_nodes(self) -> int: ...

    # PageRank shard (gdx_pr_shard_*)
    def pr_setup(self, v0: int, v1: int) -> None: ...

    def pr_init(self, contrib_slice, partials) -> None: ...

    def pr_round(self, rnd, damping, threshold, max_iter, dangling_in, contrib, contrib_slice,
                 partials) -> None: ...

    def pr_rank(self, rounds: int, rank_slice) -> None: ...

    # SSSP shard (gdx_sssp_shard_*)
    def sssp_setup(self, v0: int, v1: int) -> None: ...

    def sssp_frontier(self, dist, prev) -> int: ...

    def sssp_relax(self, dist) -> None: ...

    # optional int32 replicas (gdx_sssp_shard_*32): (count, overflow) per round
    # def sssp_frontier32(self, dist, prev) -> tuple[int, int]: ...
    # def sssp_relax32(self, dist) -> None: ...
    # and the delta exchange: the relaxation lists the vertices it lowered
    # def sssp_relax32_delta(self, dist, ids, vals) -> int: ...
    # def sssp_apply32(self, dist, ids, vals, count) -> None: ...


class DeviceExecutor:
    """Per-rank compute on this rank's GPU (libgdx.so)."""

    def __init__(self, graph):
        import torch
        self.g = graph  # paper_2401_02472_b200.DeviceGraph on cuda:LOCAL_RANK
        self._off = None
        # launch on torch's current stream so the library's kernels, NCCL
        # collectives and torch copies are stream-ordered
        graph.set_stream(torch.cuda.current_stream(graph.device).cuda_stream)

    def tc_range(self, v0, v1):
        return self.g.tc_range(v0, v1)

    def bc(self, sources):
        return self.g.bc(sources)

    def bc_into(self, sources, out):
        """gdx_bc into `out` (a device tensor is written in place)."""
        self._staged(lambda o: self.g.bc(sources, out=o), out)

    def offsets(self):
        if self._off is None:
            self._off = self.g.download().offsets
        return self._off

    def device_offsets(self, name: str):
        """offsets / rev_offsets as a device tensor (partitioning without a host copy)."""
        (t,) = self.g.device_arrays([name])
        return t

    def rev_offsets(self):
        if getattr(self, "_roff", None) is None:
            (t,) = self.g.device_arrays(["rev_offsets"])
            self._roff = t.cpu().numpy()
        return self._roff

    def num_nodes(self):
        return self.g.n

    def _staged(self, fn, *tensors):
        """Run fn on device copies of CPU tensors (collectives over gloo, e.g.
        several ranks sharing one GPU in the tests) and copy them back; CUDA
        tensors (NCCL) are passed through untouched."""
        dev = [t if t.is_cuda else t.to(f"cuda:{self.g.device}") for t in tensors]
        out = fn(*dev)
        for t, d in zip(tensors, dev):
            if d is not t:
                t.copy_(d.cpu())
        return out

    def pr_setup(self, v0, v1):
        if getattr(self, "_pr_range", None) != (v0, v1):  # the plan is cached per range
            self.g.pr_shard_setup(v0, v1)
            self._pr_range = (v0, v1)

    def pr_init(self, contrib_slice, partials):
        self._staged(self.g.pr_shard_init, contrib_slice, partials)

    def pr_round(self, rnd, damping, threshold, max_iter, dangling_in, contrib, contrib_slice,
                 partials):
        self._staged(lambda d, c, s, p: self.g.pr_shard_round(rnd, damping, threshold, max_iter,
                                                              d, c, s, p),
                     dangling_in, contrib, contrib_slice, partials)

    def pr_rank(self, rounds, rank_slice):
        self._staged(lambda r: self.g.pr_shard_rank(rounds, r), rank_slice)

    def sssp_setup(self, v0, v1):
        if getattr(self, "_sssp_range", None) != (v0, v1):
            self.g.sssp_shard_setup(v0, v1)
            self._sssp_range = (v0, v1)

    def sssp_frontier(self, dist, prev):
        return self._staged(self.g.sssp_shard_frontier, dist, prev)

    def sssp_relax(self, dist):
        self._staged(self.g.sssp_shard_relax, dist)

    def sssp_frontier32(self, dist, prev):
        return self._staged(self.g.sssp_shard_frontier32, dist, prev)

    def sssp_relax32(self, dist):
        self._staged(self.g.sssp_shard_relax32, dist)

    def sssp_relax32_delta(self, dist, ids, vals):
        return self._staged(self.g.sssp_shard_relax32_delta, dist, ids, vals)

    def sssp_apply32(self, dist, ids, vals, count):
        self._staged(lambda d, i, v: self.g.sssp_shard_apply32(d, i, v, count), dist, ids, vals)


# ---------------------------------------------------------------------------- sharded entry points

def _dist():
    import torch.distributed as dist
    return dist


def _cached_ranges(ex, kind: str, world: int, make):
    """Partitions are a pure function of the graph: computed once per executor."""
    cache = getattr(ex, "_range_cache", None)
    if cache is None:
        cache = {}
        try:
            ex._range_cache = cache
        except AttributeError:
            return make()
    key = (kind, world)
    if key not in cache:
        cache[key] = make()
    return cache[key]


def _device_for_collectives():
    import torch
    import torch.distributed as dist
    if dist.get_backend() == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def sharded_tc(ex: Executor, group=None) -> int:
    """ComputeTC across ranks: range-partitioned middle vertices + all-reduce."""
    import torch
    dist = _dist()
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    v0, v1 = _cached_ranges(ex, "tc", world, lambda: tc_ranges(ex.offsets(), world))[rank]
    local = ex.tc_range(v0, v1)
    t = torch.tensor([local], dtype=torch.int64, device=_device_for_collectives())
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return int(t.item())


def sharded_bc(ex: Executor, sources: Sequence[int], group=None, to_host: bool = True):
    """ComputeBC across ranks: source blocks + all-reduce of the partial scores
    (computed straight into the collective buffer when the executor can)."""
    import torch
    dist = _dist()
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    block = source_blocks(sources, world)[rank]
    n = ex.num_nodes()
    t = torch.zeros(n, dtype=torch.float64, device=_device_for_collectives())
    if block:
        into = getattr(ex, "bc_into", None)
        if into is not None:
            into(block, t)
        else:
            t.copy_(torch.from_numpy(np.ascontiguousarray(ex.bc(block), dtype=np.float64)))
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t.cpu().numpy() if to_host else t


def _all_gather_slices(slice_buf, ranges, out, group=None):
    """All-gather variable-length contiguous slices into `out` (padded equal
    chunks through all_gather_into_tensor, then unpacked)."""
    import torch
    dist = _dist()
    world = dist.get_world_size(group)
    chunk = slice_buf.numel()
    gathered = torch.empty(world * chunk, dtype=slice_buf.dtype, device=slice_buf.device)
    dist.all_gather_into_tensor(gathered, slice_buf, group=group)
    for r, (a, b) in enumerate(ranges):
        if b > a:
            out[a:b].copy_(gathered[r * chunk: r * chunk + (b - a)])


def balanced_ranges_device(offsets_t, parts: int) -> list[tuple[int, int]]:
    """balanced_ranges(diff(offsets) + 1, parts) computed with torch on the
    offsets' device (no host copy of the CSR)."""
    import torch
    n = offsets_t.numel() - 1
    if n <= 0:
        return [(0, 0)] * parts
    w = (offsets_t[1:] - offsets_t[:-1]).to(torch.float64) + 1.0
    csum = torch.cat([torch.zeros(1, dtype=torch.float64, device=w.device), torch.cumsum(w, 0)])
    total = csum[-1]
    t = total * torch.arange(1, parts, dtype=torch.float64, device=w.device) / parts
    cuts = [0] + torch.searchsorted(csum, t, right=False).tolist() + [n]
    cuts = np.maximum.accumulate(np.clip(np.asarray(cuts, dtype=np.int64), 0, n))
    return [(int(cuts[i]), int(cuts[i + 1])) for i in range(parts)]


def _partition(ex, kind: str, world: int):
    """Vertex ranges of `kind` ("pr": by in-edges, "sssp": by out-edges)."""
    dev = getattr(ex, "device_offsets", None)
    if dev is not None:
        return balanced_ranges_device(dev("rev_offsets" if kind == "pr" else "offsets"), world)
    if kind == "pr":
        return pr_ranges(ex.rev_offsets(), world)
    return vertex_ranges(ex.offsets(), world)


def pr_ranges(rev_offsets: np.ndarray, parts: int) -> list[tuple[int, int]]:
    """Destination-vertex ranges for PR balanced by (in-edges + vertices)."""
    indeg = np.diff(np.asarray(rev_offsets, dtype=np.int64)).astype(np.float64)
    return balanced_ranges(indeg + 1.0, parts)


def sharded_pr(ex: Executor, damping: float, threshold: float, max_iter: int, group=None,
               to_host: bool = True):
    """ComputePR across ranks -> (rank f64[n], rounds): numpy, or the
    collective-device tensor when ``to_host`` is False.  Raises
    GraphdslError("NonTermination") like gdx_pagerank when the interpreter's
    fixedPoint cap 10n+100 is hit before max_iter+1 rounds."""
    import torch
    from ._lib import GraphdslError
    dist = _dist()
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    dev = _device_for_collectives()
    n = ex.num_nodes()
    if n == 0:
        raise GraphdslError("RuntimeError", "RuntimeError: division by zero")
    ranges = _cached_ranges(ex, "pr", world, lambda: _partition(ex, "pr", world))
    v0, v1 = ranges[rank]
    chunk = max(max(b - a for a, b in ranges), 1)
    f64 = dict(dtype=torch.float64, device=dev)
    contrib = [torch.zeros(n, **f64), torch.zeros(n, **f64)]
    slice_buf = torch.zeros(chunk, **f64)
    partials = torch.zeros(2, **f64)
    ex.pr_setup(v0, v1)
    ex.pr_init(slice_buf, partials)
    _all_gather_slices(slice_buf, ranges, contrib[0], group)
    dist.all_reduce(partials, op=dist.ReduceOp.SUM, group=group)
    dangling = partials[0:1].clone()
    cap = 10 * n + 100
    want = max_iter + 1 if max_iter >= 0 else 1
    limit = min(want, cap)
    rounds = limit
    for r in range(limit):
        ex.pr_round(r, damping, threshold, max_iter, dangling, contrib[r & 1], slice_buf, partials)
        _all_gather_slices(slice_buf, ranges, contrib[(r + 1) & 1], group)
        dist.all_reduce(partials, op=dist.ReduceOp.SUM, group=group)
        dangling.copy_(partials[0:1])
        if float(partials[1].item()) == 0.0:
            rounds = r + 1
            break
    else:
        if limit < want:
            raise GraphdslError("NonTermination", f"NonTermination: fixedPoint exceeded {cap} "
                                "iterations without converging")
    rank_slice = torch.zeros(chunk, **f64)
    ex.pr_rank(rounds, rank_slice)
    out = torch.zeros(n, **f64)
    _all_gather_slices(rank_slice, ranges, out, group)
    return (out.cpu().numpy() if to_host else out), rounds


def _renumbered(ex: "DeviceExecutor", algo: str):
    """(executor over the degree-ordered renumbering gdx_pagerank / gdx_sssp
    run this graph on, newid) or None (csrc/relabel.cu).  Every rank renumbers
    its replica with the same deterministic sort, so the ranks agree on the
    ids.  The renumbered graph's handle is re-queried on every call (it is
    rebuilt when the weights change); its executor is kept while it stays the
    same handle."""
    from .graph import _BorrowedGraph
    if isinstance(ex.g, _BorrowedGraph):
        return None
    r = ex.g.renumbered(algo)
    if r is None:
        return None
    h, newid = r
    cache = ex.__dict__.setdefault("_ren", {})
    old = cache.get(algo)
    if old is None or old[0].g._h.value != h._h.value:
        cache[algo] = (DeviceExecutor(h), newid)
    else:
        h.close()
    return cache[algo][0], newid


def sharded_pr_p2p(ex: "DeviceExecutor", damping: float, threshold: float, max_iter: int,
                   group=None, to_host: bool = True):
    """ComputePR across ranks with the exchange fused into the kernels over
    peer memory (gdx_pr_p2p_*): pass B stores every new contrib value straight
    into every rank's buffer over NVLink, partials are published with
    system-scope atomics.  torch.distributed only carries the one-time IPC
    handle exchange and the final rank gather.  Same result and rounds as
    sharded_pr / gdx_pagerank."""
    import torch
    from ._lib import GraphdslError
    dist = _dist()
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    n = ex.num_nodes()
    if n == 0:
        raise GraphdslError("RuntimeError", "RuntimeError: division by zero")
    ren = _renumbered(ex, "pr")
    if ren is not None:  # the partitions of the graph gdx_pagerank runs on
        rex, newid = ren
        out, rounds = sharded_pr_p2p(rex, damping, threshold, max_iter, group, to_host=False)
        out = torch.index_select(out, 0, newid.to(out.device))
        return (out.cpu().numpy() if to_host else out), rounds
    ranges = _cached_ranges(ex, "pr", world, lambda: _partition(ex, "pr", world))
    v0, v1 = ranges[rank]
    g = ex.g
    if getattr(ex, "_p2p", None) != (world, rank, v0, v1):
        ex.pr_setup(v0, v1)
        mine = g.pr_p2p_setup(world, rank)
        allh = [None] * world
        dist.all_gather_object(allh, mine, group=group)
        g.pr_p2p_open(b"".join(allh))
        ex._p2p = (world, rank, v0, v1)
    dangling, _ = g.pr_p2p_init()
    cap = 10 * n + 100
    want = max_iter + 1 if max_iter >= 0 else 1
    limit = min(want, cap)
    rounds = limit
    # rounds in growing batches without host round trips (the same schedule
    # on every rank); rounds past the settled one exit on the device
    r, batch = 0, 4
    while r < limit:
        cnt = min(batch, limit - r)
        settled = g.pr_p2p_rounds(r, cnt, damping, threshold, max_iter, dangling)
        if settled >= 0:
            rounds = settled + 1
            break
        r += cnt
        batch = min(2 * batch, 64)
    else:
        if limit < want:
            raise GraphdslError("NonTermination", f"NonTermination: fixedPoint exceeded {cap} "
                                "iterations without converging")
    dev = _device_for_collectives()
    chunk = max(max(b - a for a, b in ranges), 1)
    # no zero fills: the slice's padding is never unpacked, and the ranges
    # cover [0, n), so every entry of `out` is written
    rank_slice = torch.empty(chunk, dtype=torch.float64, device=dev)
    ex.pr_rank(rounds, rank_slice)
    out = torch.empty(n, dtype=torch.float64, device=dev)
    _all_gather_slices(rank_slice, ranges, out, group)
    return (out.cpu().numpy() if to_host else out), rounds


INF64 = (2**63 - 1) // 2
INF32 = 2**31 - 1


def sharded_sssp(ex: Executor, src: int, group=None, to_host: bool = True, stats=None,
                 width: Optional[int] = None, exchange: Optional[str] = None):
    """ComputeSSSP across ranks -> int64[n] (INF = INT64_MAX/2), bit-exact;
    numpy, or the collective-device tensor when ``to_host`` is False.

    Rounds run over int32 replicas when the executor has them (half the
    gather and all-reduce bytes); if any rank's relaxation would reach
    INT32_MAX the call reruns over int64 replicas (``width`` forces one).
    ``exchange``: "delta" (default with int32 replicas and more than one rank)
    all-gathers only the vertices each rank lowered in the round and applies
    them with an element-wise MIN, falling back to the dense MIN all-reduce of
    the replica in rounds where the lists are not smaller; "dense" always
    all-reduces the replica."""
    import torch
    from ._lib import GraphdslError
    dist = _dist()
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    dev = _device_for_collectives()
    n = ex.num_nodes()
    if not 0 <= src < n:
        raise GraphdslError("RuntimeError", f"RuntimeError: node id {src} out of range [0, {n})")
    if exchange not in (None, "delta", "dense"):
        raise GraphdslError("InvalidArgument", f"InvalidArgument: exchange {exchange!r}")
    v0, v1 = _cached_ranges(ex, "sssp", world, lambda: _partition(ex, "sssp", world))[rank]
    ex.sssp_setup(v0, v1)
    d = None
    if width != 64 and hasattr(ex, "sssp_frontier32"):
        delta = exchange != "dense" and world > 1 and hasattr(ex, "sssp_relax32_delta")
        d32 = _sssp_rounds(ex, src, n, dev, torch.int32, group, stats, delta)
        if d32 is not None:
            d = d32.to(torch.int64)
            d[d32 == INF32] = INF64
    elif width == 32:
        raise GraphdslError("Unsupported", "Unsupported: executor has no int32 SSSP shard")
    if d is None:
        d = _sssp_rounds(ex, src, n, dev, torch.int64, group, stats, False)
    return d.cpu().numpy() if to_host else d


def sharded_sssp_p2p(ex: "DeviceExecutor", src: int, group=None, to_host: bool = True,
                     stats=None):
    """ComputeSSSP across ranks with the exchange fused into the relaxation
    over peer memory (gdx_sssp_p2p_*): vertex ranges balanced by out-edges,
    improving candidates sent to the owners' replicas by peer atomicMin, the
    round loop and its barriers on the devices -- no collective and no host
    round trip per round.  torch.distributed carries only the one-time IPC
    handle exchange.  Every rank returns the whole int64 vector (read from the
    owners' replicas); bit-exact."""
    import torch
    from ._lib import GraphdslError
    dist = _dist()
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    n = ex.num_nodes()
    if not 0 <= src < n:
        raise GraphdslError("RuntimeError", f"RuntimeError: node id {src} out of range [0, {n})")
    ren = _renumbered(ex, "sssp")
    if ren is not None:  # the partitions of the graph gdx_sssp runs on
        rex, newid = ren
        out = sharded_sssp_p2p(rex, int(newid[src].item()), group, to_host=False, stats=stats)
        out = torch.index_select(out, 0, newid.to(out.device))
        return out.cpu().numpy() if to_host else out
    ranges = _cached_ranges(ex, "sssp", world, lambda: _partition(ex, "sssp", world))
    g = ex.g
    if getattr(ex, "_sssp_p2p", None) != (world, rank, tuple(ranges)):
        bounds = [r[0] for r in ranges] + [ranges[-1][1]]
        mine = g.sssp_p2p_setup(world, rank, bounds)
        allh = [None] * world
        dist.all_gather_object(allh, mine, group=group)
        g.sssp_p2p_open(b"".join(allh))
        ex._sssp_p2p = (world, rank, tuple(ranges))
    out = torch.empty(n, dtype=torch.int64, device=f"cuda:{g.device}")
    g.sssp_p2p_run(src, out=out, stats=stats)
    return out.cpu().numpy() if to_host else out


def _sssp_rounds(ex, src, n, dev, dtype, group, stats, delta):
    """fixedPoint rounds of sharded_sssp over `dtype` replicas; None when an
    int32 relaxation overflowed on any rank."""
    import torch
    from ._lib import GraphdslError
    dist = _dist()
    world = dist.get_world_size(group)
    wide = dtype == torch.int64
    d = torch.full((n,), INF64 if wide else INF32, dtype=dtype, device=dev)
    prev = d.clone()
    d[src] = 0
    cnt = torch.zeros(2, dtype=torch.int64, device=dev)
    if delta:
        ids = torch.empty(n, dtype=torch.int32, device=dev)
        vals = torch.empty(n, dtype=torch.int32, device=dev)
    sparse_rounds = dense_rounds = 0
    cap = 10 * n + 100
    for r in range(cap + 1):
        if wide:
            cnt[0], cnt[1] = ex.sssp_frontier(d, prev), 0
        else:
            cnt[0], cnt[1] = ex.sssp_frontier32(d, prev)
        dist.all_reduce(cnt, op=dist.ReduceOp.SUM, group=group)
        c, ovf = (int(x) for x in cnt.tolist())
        if ovf:
            return None
        if c == 0:
            if stats is not None:
                stats.update(rounds=r + 1, width=64 if wide else 32,
                             exchange={"sparse_rounds": sparse_rounds, "dense_rounds": dense_rounds})
            return d
        if not delta:
            if wide:
                ex.sssp_relax(d)
            else:
                ex.sssp_relax32(d)
            if world > 1:
                dist.all_reduce(d, op=dist.ReduceOp.MIN, group=group)
                dense_rounds += 1
            continue
        k = ex.sssp_relax32_delta(d, ids, vals)
        ks = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(world)]
        dist.all_gather(ks, torch.tensor([k], dtype=torch.int64, device=dev), group=group)
        kmax = max(int(x) for x in torch.cat(ks).tolist())
        if 2 * world * kmax > n:  # the lists are not smaller than the replica
            dist.all_reduce(d, op=dist.ReduceOp.MIN, group=group)
            dense_rounds += 1
        elif kmax > 0:
            ids[k:kmax] = -1  # padding to the common length
            gi = [torch.empty(kmax, dtype=torch.int32, device=dev) for _ in range(world)]
            gv = [torch.empty(kmax, dtype=torch.int32, device=dev) for _ in range(world)]
            dist.all_gather(gi, ids[:kmax], group=group)
            dist.all_gather(gv, vals[:kmax], group=group)
            ex.sssp_apply32(d, torch.cat(gi), torch.cat(gv), world * kmax)
            sparse_rounds += 1
    raise GraphdslError("NonTermination", f"NonTermination: fixedPoint exceeded {cap} iterations")


def init_from_env(backend: Optional[str] = None) -> None:
    """torchrun-style init (MASTER_ADDR/PORT, RANK, WORLD_SIZE); NCCL when CUDA
    is present, else gloo."""
    import torch
    import torch.distributed as dist
    if dist.is_initialized():
        return
    if backend is None:
        backend = "nccl" if torch.cuda.is_available() else "gloo"
    if backend == "nccl":
        import os
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    dist.init_process_group(backend)
