"""The four corpus entry points and their contracts.

Mirrors corpus::listCorpus (reference core/src/corpus.cpp:57-106): entry
function names, argument schemas, the result property/scalar, and the
tolerance the reference's own acceptance suite checks with.
"""
from __future__ import annotations

from dataclasses import dataclass, field


@dataclass(frozen=True)
class ArgSpec:
    name: str
    kind: str  # "node", "int", "float", "bool", "node-set"


@dataclass(frozen=True)
class CorpusEntry:
    name: str
    file_name: str
    entry_function: str
    args: tuple = field(default_factory=tuple)
    oracle_id: str = ""
    result_kind: str = "property"
    result_name: str = ""
    tolerance: float = 0.0
    tolerance_is_relative: bool = False


CORPUS = (
    CorpusEntry("bc", "bc.sp", "ComputeBC", (ArgSpec("sourceSet", "node-set"),), "bc",
                "property", "bc", 1e-9, True),
    CorpusEntry("pr", "pr.sp", "ComputePR",
                (ArgSpec("damping", "float"), ArgSpec("threshold", "float"),
                 ArgSpec("maxIter", "int")), "pr", "property", "rank", 1e-6, False),
    CorpusEntry("sssp", "sssp.sp", "ComputeSSSP", (ArgSpec("src", "node"),), "sssp",
                "property", "dist", 0.0, False),
    CorpusEntry("tc", "tc.sp", "ComputeTC", (), "tc", "scalar", "triangleCount", 0.0, False),
)


def list_corpus() -> tuple:
    return CORPUS


def entry_by_name(name: str) -> CorpusEntry:
    """Accepts the short name ("sssp") or the entry function ("ComputeSSSP")."""
    for e in CORPUS:
        if name in (e.name, e.entry_function):
            return e
    from ._lib import GraphdslError
    raise GraphdslError("UnknownCorpusEntry", f"UnknownCorpusEntry: '{name}'")
