"""B200-native execution backend for the four corpus algorithms of
arXiv 2401.02472 (SSSP, PageRank, Triangle Counting, Betweenness Centrality).

The compute path is libgdx.so (hand-written sm_100a CUDA behind the C ABI in
include/gdx.h); this package is the host-side mirror of the reference's
``CsrGraph`` + ``interp::run`` interface.  There is no CPU fallback.
"""
from ._lib import GraphdslError  # noqa: F401
from .corpus import CORPUS, CorpusEntry, entry_by_name, list_corpus  # noqa: F401
from .executor import RunResult, run  # noqa: F401
from .graph import (INF_DISTANCE, Context, DeviceGraph, HostCsr, MultiGraph,  # noqa: F401
                    device_count, gen_rmat_edges, gen_uniform_edges, random_weights)

__all__ = ["GraphdslError", "CORPUS", "CorpusEntry", "entry_by_name", "list_corpus",
           "RunResult", "run", "INF_DISTANCE", "DeviceGraph", "HostCsr", "device_count",
           "gen_rmat_edges", "gen_uniform_edges", "random_weights", "Context", "MultiGraph"]
