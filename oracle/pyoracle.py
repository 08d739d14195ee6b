"""TEST INFRASTRUCTURE ONLY -- ctypes bindings for the two oracles (see __init__)."""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(_HERE, "lib", "libgdx_oracle.so")
REF_SO = os.path.join(_HERE, "_ref", "libgraphdsl_ref.so")

_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)
_f64p = C.POINTER(C.c_double)
_u8p = C.POINTER(C.c_uint8)


class OracleError(RuntimeError):
    pass


class _Csr(C.Structure):
    _fields_ = [("n", C.c_int32), ("m", C.c_int32), ("directed", C.c_int32),
                ("offsets", _i32p), ("dests", _i32p), ("weights", _i32p),
                ("rev_offsets", _i32p), ("rev_srcs", _i32p), ("rev_eid", _i32p)]


def _p(a, t=_i32p):
    return None if a is None else a.ctypes.data_as(t)


@dataclass
class HostGraph:
    """Plain CSR arrays, the layout of graphdsl::CsrGraph (csr.hpp:73-81)."""
    n: int
    m: int
    directed: bool
    offsets: np.ndarray
    dests: np.ndarray
    weights: np.ndarray
    rev_offsets: np.ndarray
    rev_srcs: np.ndarray
    rev_eid: np.ndarray

    def out_degree(self) -> np.ndarray:
        return np.diff(self.offsets)


def _csr_of(g) -> tuple[_Csr, list]:
    keep = []

    def arr(name):
        a = getattr(g, name, None)
        if a is None:
            return None
        a = np.ascontiguousarray(a, dtype=np.int32)
        keep.append(a)
        return _p(a)

    c = _Csr(int(g.n), int(g.m), int(bool(g.directed)), arr("offsets"), arr("dests"),
             arr("weights"), arr("rev_offsets"), arr("rev_srcs"), arr("rev_eid"))
    return c, keep


def _copy_view(c: _Csr) -> HostGraph:
    n, m = c.n, c.m

    def grab(ptr, k):
        if k == 0 or not ptr:
            return np.zeros(k, dtype=np.int32)
        return np.ctypeslib.as_array(ptr, shape=(k,)).copy()

    return HostGraph(n, m, bool(c.directed), grab(c.offsets, n + 1), grab(c.dests, m),
                     grab(c.weights, m), grab(c.rev_offsets, n + 1), grab(c.rev_srcs, m),
                     grab(c.rev_eid, m))


def port_available() -> bool:
    return os.path.exists(PORT_SO)


def ref_available() -> bool:
    return os.path.exists(REF_SO)


class Port:
    """Our CPU restatement (gdx_oracle.cpp)."""

    def __init__(self, path: str = PORT_SO):
        if not os.path.exists(path):
            raise OracleError(f"{path} missing: run `make -C oracle port`")
        L = self.lib = C.CDLL(path)
        L.orc_last_error.restype = C.c_char_p
        L.orc_build_from_edges.argtypes = [C.c_int32, C.c_int64, _i32p, _i32p, _i32p, C.c_int,
                                           C.POINTER(C.c_void_p)]
        L.orc_graph_from_csr.argtypes = [C.POINTER(_Csr), C.POINTER(C.c_void_p)]
        L.orc_with_random_weights.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_uint64]
        L.orc_graph_view.argtypes = [C.c_void_p, C.POINTER(_Csr)]
        L.orc_graph_free.argtypes = [C.c_void_p]
        L.orc_gen_uniform_edges.argtypes = [C.c_int32, C.c_int64, C.c_uint64, _i32p, _i32p]
        L.orc_gen_rmat_edges.argtypes = [C.c_int32, C.c_int64, C.c_uint64, C.c_double, C.c_double,
                                         C.c_double, C.c_double, _i32p, _i32p]
        L.orc_gen_rmat_ctr.argtypes = [C.c_int32, C.c_int64, C.c_uint64, C.c_double, C.c_double,
                                       C.c_double, _i32p, _i32p, C.c_int]
        L.orc_gen_uniform_ctr.argtypes = [C.c_int32, C.c_int64, C.c_uint64, _i32p, _i32p, C.c_int]
        L.orc_gen_grid_ctr.argtypes = [C.c_int32, C.c_double, C.c_uint64, _i32p, _i32p]
        L.orc_gen_grid_ctr.restype = C.c_int64
        L.orc_hash_weights.argtypes = [C.POINTER(_Csr), C.c_int32, C.c_int32, C.c_uint64, _i32p,
                                       C.c_int]
        L.orc_sssp.argtypes = [C.POINTER(_Csr), C.c_int32, _i64p]
        L.orc_pr.argtypes = [C.POINTER(_Csr), C.c_double, C.c_double, C.c_int32, _f64p, _i32p,
                             C.c_int]
        L.orc_pr_rounds.argtypes = [C.POINTER(_Csr), C.c_double, C.c_int32, _f64p, C.c_int]
        L.orc_tc.argtypes = [C.POINTER(_Csr), _i64p, C.c_int]
        L.orc_tc_range.argtypes = [C.POINTER(_Csr), C.c_int32, C.c_int32, _i64p, C.c_int]
        L.orc_tc_range_owner.argtypes = [C.POINTER(_Csr), C.c_int32, C.c_int32, _i64p, C.c_int]
        L.orc_bc.argtypes = [C.POINTER(_Csr), _i32p, C.c_int32, _f64p, C.c_int]
        L.orc_bfs_levels.argtypes = [C.POINTER(_Csr), C.c_int32, _i32p]

    def _check(self, rc):
        if rc != 0:
            raise OracleError(self.lib.orc_last_error().decode())

    # -- construction ---------------------------------------------------------
    def build_from_edges(self, n, u, v, w=None, directed=True) -> HostGraph:
        u = np.ascontiguousarray(u, dtype=np.int32)
        v = np.ascontiguousarray(v, dtype=np.int32)
        w = None if w is None else np.ascontiguousarray(w, dtype=np.int32)
        h = C.c_void_p()
        self._check(self.lib.orc_build_from_edges(n, len(u), _p(u), _p(v), _p(w), int(directed),
                                                  C.byref(h)))
        try:
            c = _Csr()
            self.lib.orc_graph_view(h, C.byref(c))
            return _copy_view(c)
        finally:
            self.lib.orc_graph_free(h)

    def with_random_weights(self, g, lo, hi, seed) -> HostGraph:
        """csr.cpp:172-195 semantics (mt19937_64, canonical-pair order)."""
        c, keep = _csr_of(g)
        h = C.c_void_p()
        self._check(self.lib.orc_graph_from_csr(C.byref(c), C.byref(h)))
        try:
            self._check(self.lib.orc_with_random_weights(h, lo, hi, seed))
            out = _Csr()
            self.lib.orc_graph_view(h, C.byref(out))
            return _copy_view(out)
        finally:
            self.lib.orc_graph_free(h)

    def gen_uniform_edges(self, nodes, edges, seed):
        u = np.empty(edges, np.int32)
        v = np.empty(edges, np.int32)
        self._check(self.lib.orc_gen_uniform_edges(nodes, edges, seed, _p(u), _p(v)))
        return u, v

    def gen_rmat_edges(self, nodes, edges, seed, a=0.57, b=0.19, c=0.19, d=0.05):
        u = np.empty(edges, np.int32)
        v = np.empty(edges, np.int32)
        self._check(self.lib.orc_gen_rmat_edges(nodes, edges, seed, a, b, c, d, _p(u), _p(v)))
        return u, v

    def gen_rmat_ctr(self, nodes, edges, seed, a=0.57, b=0.19, c=0.19, threads=0):
        u = np.empty(edges, np.int32)
        v = np.empty(edges, np.int32)
        self._check(self.lib.orc_gen_rmat_ctr(nodes, edges, seed, a, b, c, _p(u), _p(v), threads))
        return u, v

    def gen_uniform_ctr(self, nodes, edges, seed, threads=0):
        u = np.empty(edges, np.int32)
        v = np.empty(edges, np.int32)
        self._check(self.lib.orc_gen_uniform_ctr(nodes, edges, seed, _p(u), _p(v), threads))
        return u, v

    def gen_grid_ctr(self, side, keep, seed):
        k = self.lib.orc_gen_grid_ctr(side, keep, seed, None, None)
        u = np.empty(k, np.int32)
        v = np.empty(k, np.int32)
        self.lib.orc_gen_grid_ctr(side, keep, seed, _p(u), _p(v))
        return u, v

    def hash_weights(self, g, lo, hi, seed, threads=0) -> np.ndarray:
        c, keep = _csr_of(g)
        w = np.empty(g.m, np.int32)
        self.lib.orc_hash_weights(C.byref(c), lo, hi, seed, _p(w), threads)
        return w

    # -- algorithms -------------------------------------------------------------
    def sssp(self, g, src) -> np.ndarray:
        c, keep = _csr_of(g)
        out = np.empty(g.n, np.int64)
        self._check(self.lib.orc_sssp(C.byref(c), src, _p(out, _i64p)))
        return out

    def pr(self, g, damping=0.85, threshold=1e-6, max_iter=100, threads=0):
        c, keep = _csr_of(g)
        out = np.empty(g.n, np.float64)
        rounds = C.c_int32(0)
        self._check(self.lib.orc_pr(C.byref(c), damping, threshold, max_iter, _p(out, _f64p),
                                    C.byref(rounds), threads))
        return out, rounds.value

    def pr_rounds(self, g, damping, rounds, threads=0):
        c, keep = _csr_of(g)
        out = np.empty(g.n, np.float64)
        self._check(self.lib.orc_pr_rounds(C.byref(c), damping, rounds, _p(out, _f64p), threads))
        return out

    def tc(self, g, threads=0) -> int:
        c, keep = _csr_of(g)
        out = C.c_int64(0)
        self._check(self.lib.orc_tc(C.byref(c), C.byref(out), threads))
        return out.value

    def tc_range(self, g, v0, v1, threads=0) -> int:
        """gdx_tc_range's partial count (owner: middle vertex if directed, smallest if not)."""
        c, keep = _csr_of(g)
        out = C.c_int64(0)
        self._check(self.lib.orc_tc_range_owner(C.byref(c), v0, v1, C.byref(out), threads))
        return out.value

    def tc_range_middle(self, g, v0, v1, threads=0) -> int:
        """tc.sp's middle-vertex partial count (any graph)."""
        c, keep = _csr_of(g)
        out = C.c_int64(0)
        self._check(self.lib.orc_tc_range(C.byref(c), v0, v1, C.byref(out), threads))
        return out.value

    def bc(self, g, sources, threads=0) -> np.ndarray:
        c, keep = _csr_of(g)
        s = np.ascontiguousarray(sources, dtype=np.int32)
        out = np.empty(g.n, np.float64)
        self._check(self.lib.orc_bc(C.byref(c), _p(s), len(s), _p(out, _f64p), threads))
        return out

    def bfs_levels(self, g, root) -> np.ndarray:
        c, keep = _csr_of(g)
        out = np.empty(g.n, np.int32)
        self._check(self.lib.orc_bfs_levels(C.byref(c), root, _p(out)))
        return out


class Ref:
    """The reference library itself (oracle/_ref/libgraphdsl_ref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise OracleError(f"{path} missing: run `make -C oracle ref` where /root/reference exists")
        L = self.lib = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_build_from_edges.argtypes = [C.c_int32, C.c_int64, _i32p, _i32p, _i32p, C.c_int,
                                           C.POINTER(C.c_void_p)]
        L.ref_with_random_weights.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_uint64,
                                              C.POINTER(C.c_void_p)]
        L.ref_transpose.argtypes = [C.c_void_p, C.POINTER(C.c_void_p)]
        L.ref_graph_view.argtypes = [C.c_void_p, C.POINTER(_Csr)]
        L.ref_graph_free.argtypes = [C.c_void_p]
        L.ref_is_edge.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.POINTER(C.c_int)]
        L.ref_gen_uniform_edges.argtypes = [C.c_int32, C.c_int64, C.c_uint64, _i32p, _i32p]
        L.ref_gen_rmat_edges.argtypes = [C.c_int32, C.c_int64, C.c_uint64, _i32p, _i32p]
        L.ref_oracle_sssp.argtypes = [C.c_void_p, C.c_int32, _i64p]
        L.ref_oracle_pr.argtypes = [C.c_void_p, C.c_double, C.c_double, C.c_int, _f64p]
        L.ref_oracle_tc.argtypes = [C.c_void_p, C.c_int32, _i64p]
        L.ref_oracle_bc.argtypes = [C.c_void_p, _i32p, C.c_int32, _f64p]
        L.ref_oracle_bfs.argtypes = [C.c_void_p, C.c_int32, _i32p]
        L.ref_interp_sssp.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.c_int, _i64p, _u8p,
                                      C.POINTER(C.c_int)]
        L.ref_interp_pr.argtypes = [C.c_void_p, C.c_double, C.c_double, C.c_int64, C.c_int,
                                    C.c_int, _f64p, _i64p]
        L.ref_interp_tc.argtypes = [C.c_void_p, C.c_int, C.c_int, _i64p, _i64p]
        L.ref_gen_graph.argtypes = [C.c_char_p, C.c_int32, C.c_int64, C.c_uint64, C.c_char_p,
                                    C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                                    C.c_double, C.c_char_p, C.c_int]
        L.ref_interp_bc.argtypes = [C.c_void_p, _i32p, C.c_int32, C.c_int, C.c_int, _f64p]

    def _check(self, rc):
        if rc != 0:
            raise OracleError(self.lib.ref_last_error().decode())

    # Handles ---------------------------------------------------------------
    def build(self, n, u, v, w=None, directed=True) -> "RefGraph":
        u = np.ascontiguousarray(u, dtype=np.int32)
        v = np.ascontiguousarray(v, dtype=np.int32)
        w = None if w is None else np.ascontiguousarray(w, dtype=np.int32)
        h = C.c_void_p()
        self._check(self.lib.ref_build_from_edges(n, len(u), _p(u), _p(v), _p(w), int(directed),
                                                  C.byref(h)))
        return RefGraph(self, h)

    def build_from_host(self, g) -> "RefGraph":
        """Rebuild a reference CsrGraph from stored CSR arrays (CsrGraph has no
        raw-array constructor, csr.hpp:29-33): feed the canonical edges back
        through buildFromEdges, which reproduces the same arrays."""
        src = np.repeat(np.arange(g.n, dtype=np.int32), np.diff(g.offsets))
        dst = np.asarray(g.dests, dtype=np.int32)
        w = np.asarray(g.weights, dtype=np.int32)
        if not g.directed:
            keep = dst >= src
            src, dst, w = src[keep], dst[keep], w[keep]
        return self.build(g.n, src, dst, w, g.directed)

    def gen_uniform_edges(self, nodes, edges, seed):
        u = np.empty(edges, np.int32)
        v = np.empty(edges, np.int32)
        self._check(self.lib.ref_gen_uniform_edges(nodes, edges, seed, _p(u), _p(v)))
        return u, v

    def gen_rmat_edges(self, nodes, edges, seed):
        u = np.empty(edges, np.int32)
        v = np.empty(edges, np.int32)
        self._check(self.lib.ref_gen_rmat_edges(nodes, edges, seed, _p(u), _p(v)))
        return u, v

    def gen_graph_file(self, kind, nodes, edges, seed, path, weighted=False, wmin=1, wmax=100,
                       a=0.57, b=0.19, c=0.19, d=0.05) -> str:
        """graphdsl gen-graph (graphdsl.cpp:265-296): writes `path`, returns the
        summary line it prints."""
        buf = C.create_string_buffer(1024)
        self._check(self.lib.ref_gen_graph(kind.encode(), nodes, edges, seed, str(path).encode(),
                                           int(weighted), wmin, wmax, a, b, c, d, buf, 1024))
        return buf.value.decode()


class RefGraph:
    def __init__(self, ref: Ref, handle):
        self.ref, self.h = ref, handle
        c = _Csr()
        ref.lib.ref_graph_view(handle, C.byref(c))
        self.n, self.m, self.directed = c.n, c.m, bool(c.directed)

    def __del__(self):
        try:
            self.ref.lib.ref_graph_free(self.h)
        except Exception:
            pass

    def host(self) -> HostGraph:
        c = _Csr()
        self.ref.lib.ref_graph_view(self.h, C.byref(c))
        return _copy_view(c)

    def with_random_weights(self, lo, hi, seed) -> "RefGraph":
        h = C.c_void_p()
        self.ref._check(self.ref.lib.ref_with_random_weights(self.h, lo, hi, seed, C.byref(h)))
        return RefGraph(self.ref, h)

    def transpose(self) -> "RefGraph":
        h = C.c_void_p()
        self.ref._check(self.ref.lib.ref_transpose(self.h, C.byref(h)))
        return RefGraph(self.ref, h)

    def is_edge(self, u, v) -> bool:
        out = C.c_int(0)
        self.ref._check(self.ref.lib.ref_is_edge(self.h, u, v, C.byref(out)))
        return bool(out.value)

    # oracles::* ---------------------------------------------------------------
    def oracle_sssp(self, src):
        out = np.empty(self.n, np.int64)
        self.ref._check(self.ref.lib.ref_oracle_sssp(self.h, src, _p(out, _i64p)))
        return out

    def oracle_pr(self, damping, eps, max_iter):
        out = np.empty(self.n, np.float64)
        self.ref._check(self.ref.lib.ref_oracle_pr(self.h, damping, eps, max_iter, _p(out, _f64p)))
        return out

    def oracle_tc(self, max_nodes=256):
        out = C.c_int64(0)
        self.ref._check(self.ref.lib.ref_oracle_tc(self.h, max_nodes, C.byref(out)))
        return out.value

    def oracle_bc(self, sources):
        s = np.ascontiguousarray(sources, dtype=np.int32)
        out = np.empty(self.n, np.float64)
        self.ref._check(self.ref.lib.ref_oracle_bc(self.h, _p(s), len(s), _p(out, _f64p)))
        return out

    def oracle_bfs(self, root):
        out = np.empty(self.n, np.int32)
        self.ref._check(self.ref.lib.ref_oracle_bfs(self.h, root, _p(out)))
        return out

    # interp::run on the corpus ------------------------------------------------
    def interp_sssp(self, src, parallel=False, threads=4):
        dist = np.empty(self.n, np.int64)
        mod = np.empty(self.n, np.uint8)
        fin = C.c_int(0)
        self.ref._check(self.ref.lib.ref_interp_sssp(self.h, src, int(parallel), threads,
                                                     _p(dist, _i64p), _p(mod, _u8p), C.byref(fin)))
        return dist, mod, bool(fin.value)

    def interp_pr(self, damping, threshold, max_iter, parallel=False, threads=4):
        rank = np.empty(self.n, np.float64)
        it = C.c_int64(0)
        self.ref._check(self.ref.lib.ref_interp_pr(self.h, damping, threshold, max_iter,
                                                   int(parallel), threads, _p(rank, _f64p),
                                                   C.byref(it)))
        return rank, it.value

    def interp_tc(self, parallel=False, threads=4):
        cnt = C.c_int64(0)
        ret = C.c_int64(0)
        self.ref._check(self.ref.lib.ref_interp_tc(self.h, int(parallel), threads, C.byref(cnt),
                                                   C.byref(ret)))
        return cnt.value, ret.value

    def interp_bc(self, sources, parallel=False, threads=4):
        s = np.ascontiguousarray(sources, dtype=np.int32)
        out = np.empty(self.n, np.float64)
        self.ref._check(self.ref.lib.ref_interp_bc(self.h, _p(s), len(s), int(parallel), threads,
                                                   _p(out, _f64p)))
        return out
