"""Command line, after the reference's `graphdsl run` / `gen-graph`
(reference tools/graphdsl.cpp:144-158, :265-296), executing on the B200.

  python -m paper_2401_02472_b200 run sssp.sp --graph g.txt --arg src=0 [--directed]
  python -m paper_2401_02472_b200 gen-graph --kind rmat --nodes 1024 --edges 16384 --out g.txt

`run` accepts a corpus program path or entry name (sssp/pr/tc/bc or ComputeX)
and prints `name<TAB>node<TAB>value` lines for properties, `name<TAB>value`
for scalars and `return<TAB>value` (printResult, graphdsl.cpp:85-110), with
values formatted like interp::formatValue (std::to_chars shortest form).
"""
from __future__ import annotations

import argparse
import os
import sys

import numpy as np

from . import DeviceGraph, GraphdslError, entry_by_name, run

# Declaration order of the printed symbols per corpus program (parameters, then
# function-level declarations), as printResult walks the symbol table.
PRINT_ORDER = {
    "sssp": ["dist", "src", "modified", "finished"],
    "pr": ["damping", "threshold", "maxIter", "rank", "rankNext", "settled", "numNodes", "iter",
           "converged"],
    "tc": ["triangleCount"],
    "bc": ["bc"],
}


def format_value(v) -> str:
    """interp::formatValue: ints as decimal, bools true/false, doubles in the
    shortest round-trip form of std::to_chars (fixed vs scientific, shorter
    wins, ties to fixed)."""
    if isinstance(v, (bool, np.bool_)):
        return "true" if v else "false"
    if isinstance(v, (int, np.integer)):
        return str(int(v))
    x = float(v)
    if x != x:
        return "nan"
    if x in (float("inf"), float("-inf")):
        return "inf" if x > 0 else "-inf"
    if x == 0.0:
        return "-0" if np.signbit(x) else "0"
    r = repr(x)
    sign = "-" if r.startswith("-") else ""
    r = r.lstrip("-")
    if "e" in r:
        mant, exp = r.split("e")
        exp = int(exp)
    else:
        mant, exp = r, 0
    if "." in mant:
        ip, fp = mant.split(".")
    else:
        ip, fp = mant, ""
    digits = (ip + fp).lstrip("0")
    # decimal exponent of the first significant digit
    lead = len(ip.lstrip("0")) - 1 if ip.strip("0") else -(len(fp) - len(fp.lstrip("0")) + 1)
    e10 = lead + exp
    digits = digits.rstrip("0") or "0"
    sci = digits[0] + ("." + digits[1:] if len(digits) > 1 else "") + \
        f"e{'+' if e10 >= 0 else '-'}{abs(e10):02d}"
    if e10 >= 0:
        fixed = digits[:e10 + 1].ljust(e10 + 1, "0") + ("." + digits[e10 + 1:] if len(digits) > e10 + 1 else "")
    else:
        fixed = "0." + "0" * (-e10 - 1) + digits
    return sign + (fixed if len(fixed) <= len(sci) else sci)


def parse_args_kv(pairs, name: str) -> dict:
    out = {}
    for p in pairs:
        k, _, v = p.partition("=")
        if k == "sourceSet":
            out[k] = [int(t) for t in v.split(",") if t]
        elif k in ("src", "maxIter"):
            out[k] = int(v)
        else:
            out[k] = float(v)
    return out


def cmd_run(a) -> int:
    name = os.path.splitext(os.path.basename(a.program))[0]
    entry = entry_by_name(name)
    g = DeviceGraph.load_edge_list(a.graph, directed=a.directed, device=a.device)
    if a.hash_weights:
        lo, hi, seed = a.hash_weights
        g.set_hash_weights(lo, hi, seed)
    res = run(entry.name, g, parse_args_kv(a.arg, entry.name), device=a.device)
    args = parse_args_kv(a.arg, entry.name)
    lines = []
    for sym in PRINT_ORDER[entry.name]:
        if sym in res.properties:
            arr = res.properties[sym]
            boolean = arr.dtype == np.uint8
            for v, x in enumerate(arr):
                lines.append(f"{sym}\t{v}\t{format_value(bool(x) if boolean else x)}")
        elif sym in res.scalars:
            lines.append(f"{sym}\t{format_value(res.scalars[sym])}")
        elif sym in args:
            lines.append(f"{sym}\t{format_value(args[sym])}")
    if res.return_value is not None:
        lines.append(f"return\t{format_value(res.return_value)}")
    sys.stdout.write("\n".join(lines) + ("\n" if lines else ""))
    return 0


def cmd_gen(a) -> int:
    kw = dict(seed=a.seed, directed=not a.undirected, device=a.device)
    if a.weighted:
        kw["weights"] = (a.wmin, a.wmax)
    if a.kind == "grid":
        g = DeviceGraph.generate("grid", a.nodes, keep=a.keep, **kw)
    else:
        g = DeviceGraph.generate(a.kind, a.nodes, a.edges, a=a.a, b=a.b, c=a.c, **kw)
    g.write_edge_list(a.out, with_weights=a.weighted)
    print(f"wrote {a.out} (nodes {g.n}, stored edges {g.m})")
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_2401_02472_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    r = sub.add_parser("run")
    r.add_argument("program")
    r.add_argument("--graph", required=True)
    r.add_argument("--directed", action="store_true")
    r.add_argument("--arg", action="append", default=[])
    r.add_argument("--hash-weights", nargs=3, type=int, metavar=("LO", "HI", "SEED"))
    r.add_argument("--device", type=int, default=0)
    gg = sub.add_parser("gen-graph")
    gg.add_argument("--kind", choices=["rmat", "uniform", "grid"], default="rmat")
    gg.add_argument("--nodes", type=int, required=True)
    gg.add_argument("--edges", type=int, default=0)
    gg.add_argument("--seed", type=int, default=1)
    gg.add_argument("--keep", type=float, default=0.55)
    gg.add_argument("--a", type=float, default=0.57)
    gg.add_argument("--b", type=float, default=0.19)
    gg.add_argument("--c", type=float, default=0.19)
    gg.add_argument("--undirected", action="store_true")
    gg.add_argument("--weighted", action="store_true")
    gg.add_argument("--wmin", type=int, default=1)
    gg.add_argument("--wmax", type=int, default=100)
    gg.add_argument("--out", required=True)
    gg.add_argument("--device", type=int, default=0)
    a = ap.parse_args(argv)
    try:
        return cmd_run(a) if a.cmd == "run" else cmd_gen(a)
    except GraphdslError as e:
        print(f"error: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
