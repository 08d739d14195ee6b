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
    def tc_range(self, v0: int, v1: int) -> int: ...

    def bc(self, sources: Sequence[int]) -> np.ndarray: ...

    def offsets(self) -> np.ndarray: ...

    def num_nodes(self) -> int: ...


class DeviceExecutor:
    """Per-rank compute on this rank's GPU (libgdx.so)."""

    def __init__(self, graph):
        self.g = graph  # paper_2401_02472_b200.DeviceGraph on cuda:LOCAL_RANK
        self._off = None

    def tc_range(self, v0, v1):
        return self.g.tc_range(v0, v1)

    def bc(self, sources):
        return self.g.bc(sources)

    def offsets(self):
        if self._off is None:
            self._off = self.g.download().offsets
        return self._off

    def num_nodes(self):
        return self.g.n


# ---------------------------------------------------------------------------- sharded entry points

def _dist():
    import torch.distributed as dist
    return dist


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
    v0, v1 = tc_ranges(ex.offsets(), world)[rank]
    local = ex.tc_range(v0, v1)
    t = torch.tensor([local], dtype=torch.int64, device=_device_for_collectives())
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return int(t.item())


def sharded_bc(ex: Executor, sources: Sequence[int], group=None) -> np.ndarray:
    """ComputeBC across ranks: source blocks + all-reduce of the partial scores."""
    import torch
    dist = _dist()
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    block = source_blocks(sources, world)[rank]
    n = ex.num_nodes()
    part = ex.bc(block) if block else np.zeros(n, np.float64)
    t = torch.from_numpy(np.ascontiguousarray(part, dtype=np.float64)).to(_device_for_collectives())
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t.cpu().numpy()


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
