"""``run`` -- the drop-in for interp::run on the four corpus programs.

Mirrors ``graphdsl::interp::run(program, graph, args, options) -> RunResult``
(reference core/include/graphdsl/interpreter.hpp:74-88, argument binding
core/src/interpreter.cpp:1094-1148) with execution on the B200 kernels of
libgdx.so instead of the tree-walking interpreter.  The result exposes the same
symbols the interpreter leaves behind for each program:

=========  ========================================  ==================================
program    properties                                scalars / return value
=========  ========================================  ==================================
sssp       dist (int64), modified (all 0)            finished = True
pr         rank, rankNext (== rank), settled (all 1) iter, converged = True, numNodes
tc         --                                        triangleCount; returnValue
bc         bc                                        --
=========  ========================================  ==================================
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Any, Optional

import numpy as np

from ._lib import GraphdslError
from .corpus import entry_by_name
from .graph import DeviceGraph


@dataclass
class RunResult:
    properties: dict = field(default_factory=dict)
    scalars: dict = field(default_factory=dict)
    return_value: Any = None
    stats: dict = field(default_factory=dict)

    # RunResult::property / scalar (interpreter.hpp:80-81)
    def property(self, name: str) -> Optional[np.ndarray]:
        return self.properties.get(name)

    def scalar(self, name: str):
        return self.scalars.get(name)


def _as_int(v) -> int:
    # ScalarCell::store of an Int cell: Value::asInt (interpreter.hpp:26-27)
    if isinstance(v, bool):
        return 0
    if isinstance(v, float):
        return int(v)  # static_cast<int64_t>: truncation toward zero
    return int(v)


def _as_float(v) -> float:
    if isinstance(v, bool):
        return 0.0
    return float(v)


def _arg(args: dict, name: str):
    if name not in args:
        raise GraphdslError("RuntimeError", f"RuntimeError: missing argument '{name}'")
    v = args[name]
    if isinstance(v, (list, tuple, np.ndarray)):
        raise GraphdslError("RuntimeError", f"RuntimeError: argument '{name}' has the wrong shape")
    return v


def run(program: str, graph, args: Optional[dict] = None, device: int = 0) -> RunResult:
    """Execute corpus entry ``program`` ("sssp"/"ComputeSSSP", "pr", "tc", "bc")
    on ``graph`` (a DeviceGraph, or CsrGraph-like host arrays uploaded for the
    call) with interpreter-style ``args``."""
    entry = entry_by_name(program)
    bound = bind_args(entry.name, int(graph.n), dict(args or {}))
    owned = None
    if not isinstance(graph, DeviceGraph):
        owned = graph = DeviceGraph.from_csr(graph, device=device)
    try:
        res = RunResult()
        n = graph.n
        if entry.name == "sssp":
            dist = graph.sssp(bound["src"], stats=res.stats)
            res.properties = {"dist": dist, "modified": np.zeros(n, np.uint8)}
            res.scalars = {"finished": True}
        elif entry.name == "pr":
            rank, rounds = graph.pagerank(bound["damping"], bound["threshold"], bound["maxIter"],
                                          stats=res.stats)
            res.properties = {"rank": rank, "rankNext": rank.copy(),
                              "settled": np.ones(n, np.uint8)}
            res.scalars = {"iter": rounds, "converged": True, "numNodes": float(n)}
        elif entry.name == "tc":
            count = graph.tc(stats=res.stats)
            res.scalars = {"triangleCount": count}
            res.return_value = count
        else:  # bc
            res.properties = {"bc": graph.bc(bound["sourceSet"], stats=res.stats)}
        return res
    finally:
        if owned is not None:
            owned.close()


def bind_args(name: str, n: int, args: dict) -> dict:
    """Parameter binding of Machine::executeImpl (interpreter.cpp:1099-1140):
    missing / wrongly shaped arguments and out-of-range node ids raise
    RuntimeError before anything runs."""
    def node(v):
        v = _as_int(v)
        if v < 0 or v >= n:
            raise GraphdslError("RuntimeError", f"RuntimeError: node id {v} out of range [0, {n})")
        return v

    if name == "sssp":
        return {"src": node(_arg(args, "src"))}
    if name == "pr":
        max_iter = _as_int(_arg(args, "maxIter"))
        return {"damping": _as_float(_arg(args, "damping")),
                "threshold": _as_float(_arg(args, "threshold")),
                "maxIter": max(min(max_iter, 2**31 - 1), -(2**31))}
    if name == "bc":
        if "sourceSet" not in args or not isinstance(args["sourceSet"], (list, tuple, np.ndarray)):
            raise GraphdslError("RuntimeError", "RuntimeError: missing node-set argument "
                                "'sourceSet' (pass --arg sourceSet=v0,v1,...)")
        return {"sourceSet": [node(x) for x in args["sourceSet"]]}
    return {}
