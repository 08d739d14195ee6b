"""Device-resident graphs and the four entry points, over the C ABI.

``DeviceGraph`` is the B200 counterpart of the reference's immutable
``graphdsl::CsrGraph`` (core/include/graphdsl/csr.hpp:27-82): the same int32
forward + reverse CSR arrays, uploaded once and kept in HBM, with the four
corpus algorithms as methods.  ``HostCsr`` is the plain host-array layout used
to move graphs in and out (it is exactly the CsrGraph span set).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from . import _lib
from ._lib import GdxCsrView, GdxGenParams, GdxStats, GraphdslError, check

INF_DISTANCE = (2**63 - 1) // 2  # oracles.hpp:12 kInfiniteDistance


def _ptr(a) -> Optional[int]:
    """Raw address of a numpy array or torch tensor (host or device)."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):  # torch.Tensor
        if not a.is_contiguous():
            raise GraphdslError("InvalidArgument", "tensor must be contiguous")
        return a.data_ptr()
    if isinstance(a, np.ndarray):
        if not a.flags["C_CONTIGUOUS"]:
            raise GraphdslError("InvalidArgument", "array must be C-contiguous")
        return a.ctypes.data
    raise GraphdslError("InvalidArgument", f"unsupported buffer type {type(a)!r}")


def _i32(a):
    if a is None or hasattr(a, "data_ptr"):
        return a
    return np.ascontiguousarray(a, dtype=np.int32)


@dataclass
class HostCsr:
    """Host copy of the CsrGraph arrays (csr.hpp:73-81)."""
    n: int
    m: int
    directed: bool
    offsets: np.ndarray
    dests: np.ndarray
    weights: np.ndarray
    rev_offsets: np.ndarray
    rev_srcs: np.ndarray
    rev_eid: np.ndarray

    # CsrGraph-style accessors (csr.hpp:35-47)
    def node_count(self) -> int:
        return self.n

    def edge_count(self) -> int:
        return self.m

    def out_degree(self, v: int) -> int:
        return int(self.offsets[v + 1] - self.offsets[v])

    def in_degree(self, v: int) -> int:
        return int(self.rev_offsets[v + 1] - self.rev_offsets[v])

    def is_edge(self, u: int, v: int) -> bool:
        lo, hi = int(self.offsets[u]), int(self.offsets[u + 1])
        i = lo + int(np.searchsorted(self.dests[lo:hi], v))
        return i < hi and int(self.dests[i]) == v


class DeviceGraph:
    """A CSR graph resident in HBM (opaque ``gdx_graph*``)."""

    def __init__(self, handle: C.c_void_p, device: int):
        self._h = handle
        self.device = device
        n, m, d = C.c_int32(), C.c_int32(), C.c_int32()
        check(_lib.load().gdx_graph_info(handle, C.byref(n), C.byref(m), C.byref(d)))
        self.n, self.m, self.directed = n.value, m.value, bool(d.value)

    # ---- construction ---------------------------------------------------------
    @classmethod
    def from_csr(cls, g, device: int = 0) -> "DeviceGraph":
        """Upload CsrGraph arrays (numpy, or torch tensors on host or device).
        Any of weights / rev_* / dests may be None (see gdx_csr_view)."""
        lib = _lib.load()
        arrs = {k: _i32(getattr(g, k, None)) for k in
                ("offsets", "dests", "weights", "rev_offsets", "rev_srcs", "rev_eid")}
        view = GdxCsrView(int(g.n), int(g.m), int(bool(g.directed)),
                          *[_ptr(arrs[k]) for k in ("offsets", "dests", "weights", "rev_offsets",
                                                    "rev_srcs", "rev_eid")])
        h = C.c_void_p()
        check(lib.gdx_graph_create(C.byref(view), device, C.byref(h)))
        return cls(h, device)

    @classmethod
    def build_from_edges(cls, n: int, u, v, w=None, directed: bool = True,
                         device: int = 0) -> "DeviceGraph":
        """CsrGraph::buildFromEdges (csr.cpp:28-94) executed on the GPU."""
        lib = _lib.load()
        u, v, w = _i32(u), _i32(v), _i32(w)
        h = C.c_void_p()
        check(lib.gdx_graph_build_from_edges(int(n), int(len(u)), _ptr(u), _ptr(v), _ptr(w),
                                             int(bool(directed)), device, C.byref(h)))
        return cls(h, device)

    @classmethod
    def generate(cls, kind: str, nodes: int, edges: int = 0, seed: int = 1, *,
                 a: float = 0.57, b: float = 0.19, c: float = 0.19, keep: float = 0.55,
                 directed: bool = True, weights: Optional[tuple[int, int]] = None,
                 device: int = 0) -> "DeviceGraph":
        """Counter-based generators on the GPU: kind in {"rmat", "uniform", "grid"}
        (grid: ``nodes`` is the side length)."""
        lib = _lib.load()
        k = {"rmat": 0, "uniform": 1, "grid": 2}[kind]
        wlo, whi = weights if weights is not None else (1, 0)
        p = GdxGenParams(k, int(nodes), int(edges), int(seed), a, b, c, keep,
                         int(bool(directed)), int(wlo), int(whi))
        h = C.c_void_p()
        check(lib.gdx_graph_generate(C.byref(p), device, C.byref(h)))
        return cls(h, device)

    @classmethod
    def load_edge_list(cls, path: str, directed: bool = True, node_count: Optional[int] = None,
                       device: int = 0) -> "DeviceGraph":
        """CsrGraph::loadEdgeList (csr.cpp:96-130), built on the GPU."""
        h = C.c_void_p()
        check(_lib.load().gdx_graph_load_edge_list(
            str(path).encode(), int(bool(directed)), -1 if node_count is None else int(node_count),
            device, C.byref(h)))
        return cls(h, device)

    def write_edge_list(self, path: str, with_weights: bool = False) -> None:
        """writeEdgeList (csr.cpp:211-223)."""
        check(_lib.load().gdx_graph_write_edge_list(self.handle, str(path).encode(),
                                                    int(bool(with_weights))))

    def set_random_weights(self, lo: int, hi: int, seed: int) -> None:
        """CsrGraph::withRandomWeights (csr.cpp:172-195): the reference's
        mt19937_64 weights, drawn on the host side of libgdx, uploaded."""
        check(_lib.load().gdx_graph_set_random_weights(self.handle, int(lo), int(hi), int(seed)))

    def set_hash_weights(self, lo: int, hi: int, seed: int) -> None:
        check(_lib.load().gdx_graph_set_hash_weights(self._h, lo, hi, seed))

    def download(self, arrays: Optional[Sequence[str]] = None) -> HostCsr:
        """Host copy of the CSR; ``arrays`` limits it to the named arrays (the
        others are None) -- e.g. ("offsets", "dests", "weights") for a
        billion-edge graph whose reverse arrays alias the forward ones."""
        n, m = self.n, self.m
        order = ("offsets", "dests", "weights", "rev_offsets", "rev_srcs", "rev_eid")
        want = order if arrays is None else tuple(arrays)
        a = {k: (np.empty(n + 1 if "offsets" in k else m, np.int32) if k in want else None)
             for k in order}
        check(_lib.load().gdx_graph_download(self._h, *[_ptr(a[k]) for k in order]))
        return HostCsr(n, m, self.directed, **a)

    def device_arrays(self, names: Sequence[str]):
        """Device (torch, int32) copies of the named CSR arrays, for on-device
        checks at sizes where a host copy is impractical."""
        import torch
        n, m = self.n, self.m
        order = ("offsets", "dests", "weights", "rev_offsets", "rev_srcs", "rev_eid")
        out = {k: torch.empty(n + 1 if "offsets" in k else m, dtype=torch.int32,
                              device=f"cuda:{self.device}") for k in names}
        ptrs = [_ptr(out[k]) if k in out else None for k in order]
        check(_lib.load().gdx_graph_download(self._h, *ptrs))
        torch.cuda.synchronize(self.device)
        return [out[k] for k in names]

    # ---- lifetime / streams ---------------------------------------------------
    def close(self) -> None:
        if self._h:
            check(_lib.load().gdx_graph_destroy(self._h))
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def renumbered(self, algo: str):
        """The degree-ordered renumbering the library runs PageRank ("pr") /
        SSSP ("sssp") on for this graph (gdx_graph_renumbered): (the renumbered
        graph, owned by this one -- valid until this graph is closed or its
        weights change --, newid as an int32 device tensor), or None when the
        graph is not renumbered."""
        import torch
        h = C.c_void_p()
        newid = torch.empty(max(self.n, 1), dtype=torch.int32, device=f"cuda:{self.device}")
        check(_lib.load().gdx_graph_renumbered(self._h, 0 if algo == "pr" else 1, C.byref(h),
                                               _ptr(newid)))
        if not h.value:
            return None
        return _BorrowedGraph(h, self.device, self), newid[: self.n]

    def __exit__(self, *exc):
        self.close()

    @property
    def handle(self) -> C.c_void_p:
        if not self._h:
            raise GraphdslError("InvalidArgument", "graph handle is closed")
        return self._h

    def set_stream(self, stream_ptr: Optional[int]) -> None:
        """Launch on this CUDA stream (e.g. ``torch.cuda.current_stream().cuda_stream``).
        None selects the handle's own stream; 0 (torch's default stream) maps to
        cudaStreamLegacy so the library's work is ordered with torch's."""
        if stream_ptr == 0:
            stream_ptr = 1  # cudaStreamLegacy
        check(_lib.load().gdx_graph_set_stream(self.handle, stream_ptr))

    def stream(self) -> int:
        s = C.c_void_p()
        check(_lib.load().gdx_graph_get_stream(self.handle, C.byref(s)))
        return s.value or 0

    # ---- the four entry points ----------------------------------------------
    def sssp(self, src: int, out=None, stats: Optional[dict] = None):
        """ComputeSSSP -> int64 distances (INF = INT64_MAX/2).  ``out`` may be a
        host array or a device tensor of n int64."""
        res = out if out is not None else np.empty(self.n, np.int64)
        st = GdxStats()
        check(_lib.load().gdx_sssp(self.handle, int(src), _ptr(res), C.byref(st)))
        if stats is not None:
            stats.update(st.as_dict())
        return res

    def pagerank(self, damping: float = 0.85, threshold: float = 1e-6, max_iter: int = 100,
                 out=None, stats: Optional[dict] = None):
        """ComputePR -> (rank f64[n], rounds)."""
        res = out if out is not None else np.empty(self.n, np.float64)
        rounds = C.c_int32()
        st = GdxStats()
        check(_lib.load().gdx_pagerank(self.handle, float(damping), float(threshold),
                                       int(max_iter), _ptr(res), C.byref(rounds), C.byref(st)))
        if stats is not None:
            stats.update(st.as_dict())
        return res, rounds.value

    def tc(self, stats: Optional[dict] = None) -> int:
        """ComputeTC -> triangle count (tc.sp semantics)."""
        cnt = C.c_int64()
        st = GdxStats()
        check(_lib.load().gdx_tc(self.handle, C.byref(cnt), C.byref(st)))
        if stats is not None:
            stats.update(st.as_dict())
        return cnt.value

    def tc_range(self, v_begin: int, v_end: int, stats: Optional[dict] = None) -> int:
        cnt = C.c_int64()
        st = GdxStats()
        check(_lib.load().gdx_tc_range(self.handle, int(v_begin), int(v_end), C.byref(cnt),
                                       C.byref(st)))
        if stats is not None:
            stats.update(st.as_dict())
        return cnt.value

    def bc(self, sources: Sequence[int], out=None, stats: Optional[dict] = None):
        """ComputeBC -> f64[n] (unnormalised, sources excluded)."""
        src = np.ascontiguousarray(np.asarray(sources, dtype=np.int64).astype(np.int32))
        if len(src) != len(sources):
            raise GraphdslError("InvalidArgument", "bad source set")
        res = out if out is not None else np.empty(self.n, np.float64)
        st = GdxStats()
        check(_lib.load().gdx_bc(self.handle, _ptr(src) if len(src) else None, len(src),
                                 _ptr(res), C.byref(st)))
        if stats is not None:
            stats.update(st.as_dict())
        return res

    # ---- textbook kernels (oracles.cpp on the device; `check`) ------------------
    def textbook_sssp(self, src: int) -> np.ndarray:
        out = np.empty(self.n, np.int64)
        check(_lib.load().gdx_textbook_sssp(self.handle, int(src), _ptr(out)))
        return out

    def textbook_pr(self, damping: float, eps: float, max_iter: int) -> np.ndarray:
        out = np.empty(self.n, np.float64)
        check(_lib.load().gdx_textbook_pr(self.handle, float(damping), float(eps), int(max_iter),
                                          _ptr(out)))
        return out

    def textbook_tc(self) -> int:
        c = C.c_int64()
        check(_lib.load().gdx_textbook_tc(self.handle, C.byref(c)))
        return c.value

    def textbook_bc(self, sources: Sequence[int]) -> np.ndarray:
        src = np.ascontiguousarray(np.asarray(sources, dtype=np.int64).astype(np.int32))
        out = np.empty(self.n, np.float64)
        check(_lib.load().gdx_textbook_bc(self.handle, _ptr(src) if len(src) else None, len(src),
                                          _ptr(out)))
        return out

    # ---- multi-GPU shards (distributed.py drives the exchange) ------------------
    def pr_shard_setup(self, v_begin: int, v_end: int) -> None:
        check(_lib.load().gdx_pr_shard_setup(self.handle, int(v_begin), int(v_end)))

    def pr_shard_init(self, contrib_slice, partials) -> None:
        check(_lib.load().gdx_pr_shard_init(self.handle, _ptr(contrib_slice), _ptr(partials)))

    def pr_shard_round(self, rnd: int, damping: float, threshold: float, max_iter: int,
                       dangling_in, contrib_in, contrib_slice, partials) -> None:
        check(_lib.load().gdx_pr_shard_round(self.handle, int(rnd), float(damping),
                                             float(threshold), int(max_iter), _ptr(dangling_in),
                                             _ptr(contrib_in), _ptr(contrib_slice),
                                             _ptr(partials)))

    def pr_shard_rank(self, rounds: int, rank_slice) -> None:
        check(_lib.load().gdx_pr_shard_rank(self.handle, int(rounds), _ptr(rank_slice)))

    def pr_p2p_setup(self, world: int, rank: int) -> bytes:
        h = C.create_string_buffer(64)
        check(_lib.load().gdx_pr_p2p_setup(self.handle, int(world), int(rank), h))
        return h.raw

    def pr_p2p_open(self, handles: bytes) -> None:
        buf = C.create_string_buffer(handles, len(handles))
        check(_lib.load().gdx_pr_p2p_open(self.handle, buf))

    def pr_p2p_init(self) -> tuple[float, float]:
        out = (C.c_double * 2)()
        check(_lib.load().gdx_pr_p2p_init(self.handle, out))
        return out[0], out[1]

    def pr_p2p_round(self, rnd: int, damping: float, threshold: float, max_iter: int,
                     dangling_in: float) -> tuple[float, float]:
        out = (C.c_double * 2)()
        check(_lib.load().gdx_pr_p2p_round(self.handle, int(rnd), float(damping), float(threshold),
                                           int(max_iter), float(dangling_in), out))
        return out[0], out[1]

    def pr_p2p_rounds(self, first: int, count: int, damping: float, threshold: float,
                      max_iter: int, dangling_in: float) -> int:
        """Rounds [first, first+count) without host round trips -> the first
        settled round in the range, or -1."""
        st = C.c_int32(-1)
        check(_lib.load().gdx_pr_p2p_rounds(self.handle, int(first), int(count), float(damping),
                                            float(threshold), int(max_iter), float(dangling_in),
                                            C.byref(st)))
        return st.value

    def pr_p2p_close(self) -> None:
        check(_lib.load().gdx_pr_p2p_close(self.handle))

    def sssp_p2p_setup(self, world: int, rank: int, bounds: Sequence[int]) -> bytes:
        b = np.ascontiguousarray(np.asarray(bounds, dtype=np.int32))
        h = C.create_string_buffer(64)
        check(_lib.load().gdx_sssp_p2p_setup(self.handle, int(world), int(rank), _ptr(b), h))
        return h.raw

    def sssp_p2p_open(self, handles: bytes) -> None:
        buf = C.create_string_buffer(bytes(handles), len(handles))
        check(_lib.load().gdx_sssp_p2p_open(self.handle, buf))

    def sssp_p2p_run(self, src: int, out=None, stats: Optional[dict] = None):
        res = out if out is not None else np.empty(self.n, np.int64)
        st = GdxStats()
        check(_lib.load().gdx_sssp_p2p_run(self.handle, int(src), _ptr(res), C.byref(st)))
        if stats is not None:
            stats.update(st.as_dict())
        return res

    def sssp_p2p_close(self) -> None:
        check(_lib.load().gdx_sssp_p2p_close(self.handle))

    def sssp_shard_setup(self, v_begin: int, v_end: int) -> None:
        check(_lib.load().gdx_sssp_shard_setup(self.handle, int(v_begin), int(v_end)))

    def sssp_shard_frontier(self, dist, prev) -> int:
        c = np.zeros(1, np.int64)
        check(_lib.load().gdx_sssp_shard_frontier(self.handle, _ptr(dist), _ptr(prev), _ptr(c)))
        return int(c[0])

    def sssp_shard_relax(self, dist) -> None:
        check(_lib.load().gdx_sssp_shard_relax(self.handle, _ptr(dist)))

    def sssp_shard_frontier32(self, dist, prev):
        """int32 replicas (INF = INT32_MAX) -> (improved count, overflow flag)."""
        c = np.zeros(2, np.int64)
        check(_lib.load().gdx_sssp_shard_frontier32(self.handle, _ptr(dist), _ptr(prev), _ptr(c)))
        return int(c[0]), int(c[1])

    def sssp_shard_relax32(self, dist) -> None:
        check(_lib.load().gdx_sssp_shard_relax32(self.handle, _ptr(dist)))

    def sssp_shard_relax32_delta(self, dist, ids, vals) -> int:
        """int32 relaxation listing the vertices it lowered (ids, their values)
        -> how many."""
        c = np.zeros(1, np.int64)
        check(_lib.load().gdx_sssp_shard_relax32_delta(self.handle, _ptr(dist), _ptr(ids),
                                                       _ptr(vals), _ptr(c)))
        return int(c[0])

    def sssp_shard_apply32(self, dist, ids, vals, count: int) -> None:
        check(_lib.load().gdx_sssp_shard_apply32(self.handle, _ptr(dist), _ptr(ids), _ptr(vals),
                                                 int(count)))

    # ---- measurement -----------------------------------------------------------
    def profile(self, enable: bool = True) -> None:
        check(_lib.load().gdx_profile_enable(self.handle, int(enable)))

    def profile_reset(self) -> None:
        check(_lib.load().gdx_profile_reset(self.handle))

    def profile_read(self) -> dict:
        """{kernel: (total_ms, launches)} since the last reset."""
        lib = _lib.load()
        cnt = C.c_int32()
        check(lib.gdx_profile_read(self.handle, None, None, None, 0, C.byref(cnt)))
        k = cnt.value
        names = C.create_string_buffer(64 * max(k, 1))
        ms = (C.c_double * max(k, 1))()
        ln = (C.c_int64 * max(k, 1))()
        check(lib.gdx_profile_read(self.handle, names, ms, ln, k, C.byref(cnt)))
        out = {}
        for i in range(k):
            nm = names.raw[64 * i:64 * (i + 1)].split(b"\0", 1)[0].decode()
            out[nm] = (ms[i], ln[i])
        return out


def _prefer_torch_nccl() -> None:
    """libgdx dlopens NCCL for gdx_context; in a process that also uses torch it
    must be torch's bundled copy (the first libnccl.so.2 loaded wins the
    soname, and torch needs its own version's symbols)."""
    import os
    if os.environ.get("GDX_NCCL_LIB"):
        return
    try:
        import nvidia.nccl as nn
        for base in list(nn.__path__):
            p = os.path.join(base, "lib", "libnccl.so.2")
            if os.path.exists(p):
                os.environ["GDX_NCCL_LIB"] = p
                return
    except Exception:
        pass



class _BorrowedGraph(DeviceGraph):
    """A graph handle owned by another DeviceGraph (its renumbering): never
    destroyed from here."""

    def __init__(self, handle: C.c_void_p, device: int, owner: DeviceGraph):
        super().__init__(handle, device)
        self._owner = owner

    def close(self) -> None:
        self._h = None


class Context:
    """Several GPUs driven from this process (gdx_context: peer access between
    every pair, one NCCL communicator per distinct device)."""

    def __init__(self, devices: Sequence[int]):
        _prefer_torch_nccl()
        devs = (C.c_int * len(devices))(*[int(d) for d in devices])
        self._h = C.c_void_p()
        check(_lib.load().gdx_context_create(len(devices), devs, C.byref(self._h)))
        self.devices = [int(d) for d in devices]

    def info(self) -> dict:
        nd, nc, pa = C.c_int32(), C.c_int32(), C.c_int32()
        check(_lib.load().gdx_context_info(self._h, C.byref(nd), C.byref(nc), C.byref(pa)))
        return {"devices": nd.value, "nccl_comms": nc.value, "peer_access": bool(pa.value)}

    def close(self) -> None:
        if self._h:
            check(_lib.load().gdx_context_destroy(self._h))
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class MultiGraph:
    """A CsrGraph replicated on every device of a Context; the four entry
    points partitioned across the devices (gdx_*_multi)."""

    def __init__(self, ctx: Context, g):
        self.ctx = ctx  # keeps the context alive
        arrs = {k: _i32(getattr(g, k, None)) for k in
                ("offsets", "dests", "weights", "rev_offsets", "rev_srcs", "rev_eid")}
        view = GdxCsrView(int(g.n), int(g.m), int(bool(g.directed)),
                          *[_ptr(arrs[k]) for k in ("offsets", "dests", "weights", "rev_offsets",
                                                    "rev_srcs", "rev_eid")])
        self._h = C.c_void_p()
        check(_lib.load().gdx_multi_graph_create(ctx._h, C.byref(view), C.byref(self._h)))
        self.n, self.m, self.directed = int(g.n), int(g.m), bool(g.directed)

    def close(self) -> None:
        if self._h:
            check(_lib.load().gdx_multi_graph_destroy(self._h))
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def sssp(self, src: int, out=None, stats: Optional[dict] = None):
        res = out if out is not None else np.empty(self.n, np.int64)
        st = GdxStats()
        check(_lib.load().gdx_sssp_multi(self._h, int(src), _ptr(res), C.byref(st)))
        if stats is not None:
            stats.update(st.as_dict())
        return res

    def pagerank(self, damping: float = 0.85, threshold: float = 1e-6, max_iter: int = 100,
                 out=None, stats: Optional[dict] = None):
        res = out if out is not None else np.empty(self.n, np.float64)
        rounds = C.c_int32()
        st = GdxStats()
        check(_lib.load().gdx_pagerank_multi(self._h, float(damping), float(threshold),
                                             int(max_iter), _ptr(res), C.byref(rounds),
                                             C.byref(st)))
        if stats is not None:
            stats.update(st.as_dict())
        return res, rounds.value

    def tc(self, stats: Optional[dict] = None) -> int:
        cnt = C.c_int64()
        st = GdxStats()
        check(_lib.load().gdx_tc_multi(self._h, C.byref(cnt), C.byref(st)))
        if stats is not None:
            stats.update(st.as_dict())
        return cnt.value

    def bc(self, sources: Sequence[int], out=None, stats: Optional[dict] = None):
        src = np.ascontiguousarray(np.asarray(sources, dtype=np.int64).astype(np.int32))
        res = out if out is not None else np.empty(self.n, np.float64)
        st = GdxStats()
        check(_lib.load().gdx_bc_multi(self._h, _ptr(src) if len(src) else None, len(src),
                                       _ptr(res), C.byref(st)))
        if stats is not None:
            stats.update(st.as_dict())
        return res


def gen_uniform_edges(nodes: int, edges: int, seed: int):
    """genUniformEdges (graphgen.cpp:8-16): the reference's edge stream."""
    u = np.empty(int(edges), np.int32)
    v = np.empty(int(edges), np.int32)
    check(_lib.load().gdx_gen_uniform_edges_ref(int(nodes), int(edges), int(seed), _ptr(u), _ptr(v)))
    return u, v


def gen_rmat_edges(nodes: int, edges: int, seed: int, a: float = 0.57, b: float = 0.19,
                   c: float = 0.19, d: float = 0.05):
    """genRmatEdges (graphgen.cpp:18-56): the reference's edge stream."""
    u = np.empty(int(edges), np.int32)
    v = np.empty(int(edges), np.int32)
    check(_lib.load().gdx_gen_rmat_edges_ref(int(nodes), int(edges), int(seed), a, b, c, d,
                                             _ptr(u), _ptr(v)))
    return u, v


def gen_edge_weights(count: int, seed: int, wmin: int, wmax: int) -> np.ndarray:
    """gen-graph's weight column (graphdsl.cpp:281-287)."""
    w = np.empty(int(count), np.int32)
    check(_lib.load().gdx_gen_edge_weights_ref(int(count), int(seed), int(wmin), int(wmax),
                                               _ptr(w)))
    return w


def random_weights(g, lo: int, hi: int, seed: int) -> np.ndarray:
    """withRandomWeights (csr.cpp:172-195) over host CSR arrays."""
    off = np.ascontiguousarray(g.offsets, np.int32)
    dst = np.ascontiguousarray(g.dests, np.int32)
    w = np.empty(int(g.m), np.int32)
    check(_lib.load().gdx_random_weights_host(int(g.n), int(g.m), int(bool(g.directed)),
                                              _ptr(off), _ptr(dst), int(lo), int(hi), int(seed),
                                              _ptr(w)))
    return w


def device_count() -> int:
    c = C.c_int()
    check(_lib.load().gdx_device_count(C.byref(c)))
    return c.value
