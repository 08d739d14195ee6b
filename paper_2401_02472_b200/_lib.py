"""ctypes binding of the C ABI (include/gdx.h) exported by lib/libgdx.so.

The product path is the CUDA library only: if libgdx.so is missing or cannot
find a GPU, calls fail loudly -- there is no CPU fallback anywhere in this
package.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libgdx.so")

i32p = C.POINTER(C.c_int32)
i64p = C.POINTER(C.c_int64)
f64p = C.POINTER(C.c_double)

# gdx_status -> CompileError-style kind (reference diagnostics.hpp:31-57)
STATUS_NAMES = {
    0: "OK", 1: "InvalidArgument", 2: "RuntimeError", 3: "RuntimeError", 4: "NonTermination",
    5: "CudaError", 6: "OutOfMemory", 7: "Unsupported", 8: "NcclError",
}


class GraphdslError(RuntimeError):
    """Mirror of graphdsl::CompileError: ``kind`` + message.  Raised for every
    non-zero gdx_status; ``kind`` is the prefix of gdx_last_error() (e.g.
    RuntimeError, NonTermination, InvalidEdge, NegativeWeight)."""

    def __init__(self, kind: str, message: str, status: int = 0):
        super().__init__(message)
        self.kind = kind
        self.status = status


class GdxCsrView(C.Structure):
    _fields_ = [("n", C.c_int32), ("m", C.c_int32), ("directed", C.c_int32),
                ("offsets", C.c_void_p), ("dests", C.c_void_p), ("weights", C.c_void_p),
                ("rev_offsets", C.c_void_p), ("rev_srcs", C.c_void_p), ("rev_eid", C.c_void_p)]


class GdxStats(C.Structure):
    _fields_ = [("rounds", C.c_int32), ("launches", C.c_int32), ("vertices_visited", C.c_int64),
                ("edges_visited", C.c_int64), ("updates", C.c_int64),
                ("algorithmic_bytes", C.c_double)]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


class GdxGenParams(C.Structure):
    _fields_ = [("kind", C.c_int32), ("nodes", C.c_int32), ("edges", C.c_int64),
                ("seed", C.c_uint64), ("a", C.c_double), ("b", C.c_double), ("c", C.c_double),
                ("keep", C.c_double), ("directed", C.c_int32), ("wlo", C.c_int32),
                ("whi", C.c_int32)]


# Every symbol include/gdx.h declares, with its ctypes signature.
SIGNATURES = {
    "gdx_last_error": ([], C.c_char_p),
    "gdx_abi_version": ([], C.c_int),
    "gdx_device_count": ([C.POINTER(C.c_int)], C.c_int),
    "gdx_graph_create": ([C.POINTER(GdxCsrView), C.c_int, C.POINTER(C.c_void_p)], C.c_int),
    "gdx_graph_destroy": ([C.c_void_p], C.c_int),
    "gdx_pool_trim": ([i64p], C.c_int),
    "gdx_graph_info": ([C.c_void_p, i32p, i32p, i32p], C.c_int),
    "gdx_graph_download": ([C.c_void_p] + [C.c_void_p] * 6, C.c_int),
    "gdx_graph_set_stream": ([C.c_void_p, C.c_void_p], C.c_int),
    "gdx_graph_get_stream": ([C.c_void_p, C.POINTER(C.c_void_p)], C.c_int),
    "gdx_graph_build_from_edges": ([C.c_int32, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p,
                                    C.c_int, C.c_int, C.POINTER(C.c_void_p)], C.c_int),
    "gdx_graph_load_edge_list": ([C.c_char_p, C.c_int, C.c_int32, C.c_int,
                                  C.POINTER(C.c_void_p)], C.c_int),
    "gdx_graph_write_edge_list": ([C.c_void_p, C.c_char_p, C.c_int], C.c_int),
    "gdx_graph_generate": ([C.POINTER(GdxGenParams), C.c_int, C.POINTER(C.c_void_p)], C.c_int),
    "gdx_graph_set_hash_weights": ([C.c_void_p, C.c_int32, C.c_int32, C.c_uint64], C.c_int),
    "gdx_gen_uniform_edges_ref": ([C.c_int32, C.c_int64, C.c_uint64, C.c_void_p, C.c_void_p],
                                  C.c_int),
    "gdx_gen_rmat_edges_ref": ([C.c_int32, C.c_int64, C.c_uint64, C.c_double, C.c_double,
                               C.c_double, C.c_double, C.c_void_p, C.c_void_p], C.c_int),
    "gdx_gen_edge_weights_ref": ([C.c_int64, C.c_uint64, C.c_int32, C.c_int32, C.c_void_p],
                                 C.c_int),
    "gdx_random_weights_host": ([C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p,
                                C.c_int32, C.c_int32, C.c_uint64, C.c_void_p], C.c_int),
    "gdx_graph_set_random_weights": ([C.c_void_p, C.c_int32, C.c_int32, C.c_uint64], C.c_int),
    "gdx_sssp": ([C.c_void_p, C.c_int32, C.c_void_p, C.POINTER(GdxStats)], C.c_int),
    "gdx_pagerank": ([C.c_void_p, C.c_double, C.c_double, C.c_int32, C.c_void_p, i32p,
                      C.POINTER(GdxStats)], C.c_int),
    "gdx_tc": ([C.c_void_p, i64p, C.POINTER(GdxStats)], C.c_int),
    "gdx_tc_range": ([C.c_void_p, C.c_int32, C.c_int32, i64p, C.POINTER(GdxStats)], C.c_int),
    "gdx_bc": ([C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.POINTER(GdxStats)], C.c_int),
    "gdx_pr_shard_setup": ([C.c_void_p, C.c_int32, C.c_int32], C.c_int),
    "gdx_pr_shard_init": ([C.c_void_p, C.c_void_p, C.c_void_p], C.c_int),
    "gdx_pr_shard_round": ([C.c_void_p, C.c_int32, C.c_double, C.c_double, C.c_int32,
                            C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p], C.c_int),
    "gdx_pr_shard_rank": ([C.c_void_p, C.c_int32, C.c_void_p], C.c_int),
    "gdx_pr_p2p_setup": ([C.c_void_p, C.c_int32, C.c_int32, C.c_void_p], C.c_int),
    "gdx_pr_p2p_open": ([C.c_void_p, C.c_void_p], C.c_int),
    "gdx_pr_p2p_init": ([C.c_void_p, f64p], C.c_int),
    "gdx_pr_p2p_round": ([C.c_void_p, C.c_int32, C.c_double, C.c_double, C.c_int32, C.c_double,
                          f64p], C.c_int),
    "gdx_pr_p2p_rounds": ([C.c_void_p, C.c_int32, C.c_int32, C.c_double, C.c_double, C.c_int32,
                           C.c_double, C.c_void_p], C.c_int),
    "gdx_pr_p2p_close": ([C.c_void_p], C.c_int),
    "gdx_sssp_shard_setup": ([C.c_void_p, C.c_int32, C.c_int32], C.c_int),
    "gdx_sssp_shard_frontier": ([C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p], C.c_int),
    "gdx_sssp_shard_relax": ([C.c_void_p, C.c_void_p], C.c_int),
    "gdx_sssp_shard_frontier32": ([C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p], C.c_int),
    "gdx_sssp_shard_relax32": ([C.c_void_p, C.c_void_p], C.c_int),
    "gdx_sssp_shard_relax32_delta": ([C.c_void_p] + [C.c_void_p] * 4, C.c_int),
    "gdx_sssp_shard_apply32": ([C.c_void_p] + [C.c_void_p] * 3 + [C.c_int64], C.c_int),
    "gdx_textbook_sssp": ([C.c_void_p, C.c_int32, C.c_void_p], C.c_int),
    "gdx_textbook_pr": ([C.c_void_p, C.c_double, C.c_double, C.c_int32, C.c_void_p], C.c_int),
    "gdx_textbook_tc": ([C.c_void_p, i64p], C.c_int),
    "gdx_textbook_bc": ([C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p], C.c_int),
    "gdx_context_create": ([C.c_int, C.c_void_p, C.POINTER(C.c_void_p)], C.c_int),
    "gdx_context_destroy": ([C.c_void_p], C.c_int),
    "gdx_context_info": ([C.c_void_p, i32p, i32p, i32p], C.c_int),
    "gdx_multi_graph_create": ([C.c_void_p, C.POINTER(GdxCsrView), C.POINTER(C.c_void_p)],
                               C.c_int),
    "gdx_multi_graph_destroy": ([C.c_void_p], C.c_int),
    "gdx_sssp_multi": ([C.c_void_p, C.c_int32, C.c_void_p, C.POINTER(GdxStats)], C.c_int),
    "gdx_pagerank_multi": ([C.c_void_p, C.c_double, C.c_double, C.c_int32, C.c_void_p, i32p,
                            C.POINTER(GdxStats)], C.c_int),
    "gdx_tc_multi": ([C.c_void_p, i64p, C.POINTER(GdxStats)], C.c_int),
    "gdx_bc_multi": ([C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.POINTER(GdxStats)],
                     C.c_int),
    "gdx_sssp_p2p_setup": ([C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p], C.c_int),
    "gdx_sssp_p2p_open": ([C.c_void_p, C.c_void_p], C.c_int),
    "gdx_sssp_p2p_run": ([C.c_void_p, C.c_int32, C.c_void_p, C.POINTER(GdxStats)], C.c_int),
    "gdx_sssp_p2p_close": ([C.c_void_p], C.c_int),
    "gdx_profile_enable": ([C.c_void_p, C.c_int], C.c_int),
    "gdx_graph_renumbered": ([C.c_void_p, C.c_int32, C.POINTER(C.c_void_p), C.c_void_p], C.c_int),
    "gdx_profile_reset": ([C.c_void_p], C.c_int),
    "gdx_profile_read": ([C.c_void_p, C.c_char_p, f64p, i64p, C.c_int32, i32p], C.c_int),
}

_lock = threading.Lock()
_lib = None


def load(path: str = LIB_PATH) -> C.CDLL:
    """Load libgdx.so (once).  Raises loudly when it has not been built."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise GraphdslError("Unsupported", f"{path} is missing: build it with "
                                "`python -c 'import __graft_entry__ as g; g.build()'` "
                                "or `make -C paper_2401_02472_b200/csrc`")
        lib = C.CDLL(path)
        for name, (args, res) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        _lib = lib
        return lib


def check(rc: int) -> None:
    if rc != 0:
        msg = load().gdx_last_error().decode(errors="replace")
        kind = msg.split(":", 1)[0] if ":" in msg else STATUS_NAMES.get(rc, "RuntimeError")
        raise GraphdslError(kind, msg, rc)
