"""CPU: the C-ABI library loads and exports every symbol include/gdx.h declares;
host-side argument binding mirrors interp::run (no GPU compute calls)."""
from __future__ import annotations

import ctypes
import os
import re

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "gdx.h")


def declared_symbols() -> set:
    text = open(HEADER).read()
    return set(re.findall(r"^\s*(?:const\s+)?\w+\*?\s+\*?(gdx_\w+)\s*\(", text, re.M))


def test_header_declares_entry_points():
    syms = declared_symbols()
    for s in ("gdx_graph_create", "gdx_sssp", "gdx_pagerank", "gdx_tc", "gdx_bc",
              "gdx_graph_build_from_edges", "gdx_last_error"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    from paper_2401_02472_b200 import _lib
    lib = _lib.load()
    syms = declared_symbols()
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    # the Python binding covers exactly the declared ABI
    assert set(_lib.SIGNATURES) == syms
    assert lib.gdx_abi_version() == 1


def test_library_is_sm100a_only():
    so = os.path.join(ROOT, "paper_2401_02472_b200", "lib", "libgdx.so")
    data = open(so, "rb").read()
    assert b"sm_100a" in data


def test_no_cpu_fallback_without_gpu():
    """The product path fails loudly where no GPU is visible."""
    import paper_2401_02472_b200 as gdx
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if has_gpu:
        pytest.skip("GPU present")
    with pytest.raises(gdx.GraphdslError) as e:
        gdx.device_count()
    assert e.value.kind == "CudaError"


def test_bind_args_mirrors_interpreter(known):
    from paper_2401_02472_b200 import GraphdslError
    from paper_2401_02472_b200.executor import bind_args
    err = known["errors"]
    with pytest.raises(GraphdslError) as e:
        bind_args("sssp", 3, {"src": 99})
    assert str(e.value) == err["sssp_src_out_of_range"] and e.value.kind == "RuntimeError"
    with pytest.raises(GraphdslError) as e:
        bind_args("bc", 3, {"sourceSet": [0, 7]})
    assert str(e.value) == err["bc_source_out_of_range"]
    with pytest.raises(GraphdslError, match="missing argument 'src'"):
        bind_args("sssp", 3, {})
    with pytest.raises(GraphdslError, match="missing node-set argument 'sourceSet'"):
        bind_args("bc", 3, {})
    with pytest.raises(GraphdslError, match="wrong shape"):
        bind_args("pr", 3, {"damping": [1], "threshold": 0.1, "maxIter": 3})
    b = bind_args("pr", 3, {"damping": 0.85, "threshold": 1e-9, "maxIter": 3.7})
    assert b["maxIter"] == 3  # static_cast<int64_t> truncation
    assert bind_args("tc", 3, {}) == {}


def test_corpus_registry():
    from paper_2401_02472_b200 import entry_by_name, list_corpus
    names = {e.entry_function for e in list_corpus()}
    assert names == {"ComputeBC", "ComputePR", "ComputeSSSP", "ComputeTC"}
    assert entry_by_name("ComputePR").result_name == "rank"
    assert entry_by_name("tc").result_kind == "scalar"
    assert entry_by_name("bc").tolerance == 1e-9 and entry_by_name("bc").tolerance_is_relative
    with pytest.raises(Exception, match="UnknownCorpusEntry"):
        entry_by_name("nope")
