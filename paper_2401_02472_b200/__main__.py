"""Command line, after the reference's `graphdsl run` / `check` / `gen-graph`
(reference tools/graphdsl.cpp:144-296, options :315-376), executing on the B200.

  python -m paper_2401_02472_b200 run sssp.sp --graph g.txt --arg src=0 [--directed]
        [--weight-min LO --weight-max HI --weight-seed S]
  python -m paper_2401_02472_b200 check pr.sp --graph g.txt [--arg ...] [--oracle pr]
  python -m paper_2401_02472_b200 gen-graph --kind rmat --nodes 1024 --edges 16384 --out g.txt
        [--weighted --weight-min 1 --weight-max 100] [--rmat-a .57 ...]

`run` accepts a corpus program path or entry name (sssp/pr/tc/bc or ComputeX)
and prints `name<TAB>node<TAB>value` lines for properties, `name<TAB>value`
for scalars and `return<TAB>value` (printResult, graphdsl.cpp:85-110), with
values formatted like interp::formatValue (std::to_chars shortest form).
`--weight-*` reassigns weights exactly like CsrGraph::withRandomWeights
(csr.cpp:172-195; drawn by libgdx's host-side copy of the reference stream).

`check` runs the device fast path, then the textbook kernels (oracles.cpp on
the device, textbook.cu), and prints the reference's comparison lines and
PASS/FAIL at the corpus tolerance (exit code 0 / 1).

`gen-graph` writes the reference's file: the genUniformEdges / genRmatEdges
edge stream in generation order, weights from the reference's
mt19937_64(seed ^ 0x9e3779b97f4a7c15) stream, then prints the undirected
summary line (graphdsl.cpp:265-296).  `--counter` selects the counter-based
device generators instead (any scale, and `--kind grid`).
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


def load_graph(a):
    g = DeviceGraph.load_edge_list(a.graph, directed=a.directed, device=a.device)
    # graphdsl.cpp:148-149 -- reassign weights when lo >= 0 and hi >= lo
    if getattr(a, "weight_min", -1) >= 0 and a.weight_max >= a.weight_min:
        g.set_random_weights(a.weight_min, a.weight_max, a.weight_seed)
    if getattr(a, "hash_weights", None):
        lo, hi, seed = a.hash_weights
        g.set_hash_weights(lo, hi, seed)
    return g


def cmd_run(a) -> int:
    if a.fp_cap:
        raise GraphdslError("Unsupported", "Unsupported: --fp-cap (the device path applies the "
                            "interpreter's default cap 10n+100)")
    name = os.path.splitext(os.path.basename(a.program))[0]
    entry = entry_by_name(name)
    g = load_graph(a)
    args = parse_args_kv(a.arg, entry.name)
    res = run(entry.name, g, args, device=a.device)
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


def _g(x: float) -> str:
    """std::ostream << double with the default precision (6, %g)."""
    return format(float(x), "g")


def cmd_check(a) -> int:
    """runCheck (graphdsl.cpp:175-256) with the device as the executor and the
    textbook kernels as the oracle."""
    name = a.oracle or os.path.splitext(os.path.basename(a.program))[0]
    entry = entry_by_name(name)
    g = load_graph(a)
    args = parse_args_kv(a.arg, entry.name)
    # per-algorithm defaults (graphdsl.cpp:187-197)
    if entry.oracle_id == "sssp":
        args.setdefault("src", 0)
    if entry.oracle_id == "bc":
        args.setdefault("sourceSet", list(range(g.n)))
    if entry.oracle_id == "pr":
        args.setdefault("damping", 0.85)
        args.setdefault("threshold", 1e-9)
        args.setdefault("maxIter", 110)
    res = run(entry.name, g, args, device=a.device)
    out = sys.stdout
    if entry.oracle_id == "tc":
        expected = g.textbook_tc()
        got = int(res.scalars["triangleCount"])
        passed = expected == got
        out.write(f"tc: device {got} oracle {expected}\n")
    elif entry.oracle_id == "sssp":
        expected = g.textbook_sssp(int(args["src"]))
        worst = int(np.max(np.abs(expected - res.properties["dist"]))) if g.n else 0
        passed = worst == 0
        out.write(f"sssp: max absolute distance error {worst}\n")
    elif entry.oracle_id == "bc":
        expected = g.textbook_bc(args["sourceSet"])
        got = res.properties["bc"]
        abs_err = float(np.max(np.abs(expected - got))) if g.n else 0.0
        scale = np.maximum(np.maximum(np.abs(expected), np.abs(got)), 1e-12)
        rel_err = float(np.max(np.abs(expected - got) / scale)) if g.n else 0.0
        passed = rel_err <= entry.tolerance
        out.write(f"bc: max abs error {_g(abs_err)}, max rel error {_g(rel_err)}\n")
    else:
        expected = g.textbook_pr(float(args["damping"]), float(args["threshold"]),
                                 int(args["maxIter"]))
        abs_err = float(np.max(np.abs(expected - res.properties["rank"]))) if g.n else 0.0
        passed = abs_err <= entry.tolerance
        out.write(f"pr: max abs error {_g(abs_err)}\n")
    tol = "exact" if entry.tolerance == 0 else \
        f"{_g(entry.tolerance)} {'relative' if entry.tolerance_is_relative else 'absolute'}"
    out.write(f"{'PASS' if passed else 'FAIL'} (tolerance {tol})\n")
    return 0 if passed else 1


def cmd_gen(a) -> int:
    from . import gen_rmat_edges, gen_uniform_edges
    if a.counter or a.kind == "grid":
        kw = dict(seed=a.seed, directed=not a.undirected, device=a.device)
        if a.weighted:
            kw["weights"] = (a.weight_min, a.weight_max)
        if a.kind == "grid":
            g = DeviceGraph.generate("grid", a.nodes, keep=a.keep, **kw)
        else:
            g = DeviceGraph.generate(a.kind, a.nodes, a.edges, a=a.rmat_a, b=a.rmat_b,
                                     c=a.rmat_c, **kw)
        g.write_edge_list(a.out, with_weights=a.weighted)
        print(f"wrote {a.out} (nodes {g.n}, stored edges {g.m})")
        return 0
    # the reference's file (graphdsl.cpp:265-296)
    if a.kind == "uniform":
        u, v = gen_uniform_edges(a.nodes, a.edges, a.seed)
    else:
        u, v = gen_rmat_edges(a.nodes, a.edges, a.seed, a.rmat_a, a.rmat_b, a.rmat_c, a.rmat_d)
    cols = [u, v]
    if a.weighted:
        from .graph import gen_edge_weights
        cols.append(gen_edge_weights(len(u), a.seed, a.weight_min, a.weight_max))
    with open(a.out, "w") as f:
        f.write(f"# {a.kind} graph: nodes {a.nodes} edges {a.edges} seed {a.seed}\n")
        if len(u):
            np.savetxt(f, np.column_stack(cols), fmt="%d", delimiter=" ")
    g = DeviceGraph.build_from_edges(a.nodes, u, v, None, directed=False, device=a.device)
    h = g.download(("offsets",))
    deg = np.diff(h.offsets)
    avg = g.m / g.n if g.n else 0.0
    print(f"wrote {a.out} (nodes {g.n}, stored edges {g.m}, avg degree {_g(avg)}, "
          f"max degree {int(deg.max()) if g.n else 0})")
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_2401_02472_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    for nm in ("run", "check"):
        r = sub.add_parser(nm)
        r.add_argument("program")
        r.add_argument("--graph", required=True)
        r.add_argument("--directed", action="store_true")
        r.add_argument("--arg", action="append", default=[])
        r.add_argument("--mode", default="seq", help="accepted for compatibility (device path)")
        r.add_argument("--threads", type=int, default=4, help="accepted for compatibility")
        r.add_argument("--device", type=int, default=0)
        if nm == "run":
            r.add_argument("--fp-cap", type=int, default=0)
            r.add_argument("--weight-min", type=int, default=-1)
            r.add_argument("--weight-max", type=int, default=-1)
            r.add_argument("--weight-seed", type=int, default=1)
            r.add_argument("--hash-weights", nargs=3, type=int, metavar=("LO", "HI", "SEED"),
                           help="counter-hash weights (device generator; not the reference's)")
        else:
            r.add_argument("--oracle", default="")
    gg = sub.add_parser("gen-graph")
    gg.add_argument("--kind", choices=["rmat", "uniform", "grid"], default="uniform")
    gg.add_argument("--nodes", type=int, default=1024)
    gg.add_argument("--edges", type=int, default=8192)
    gg.add_argument("--seed", type=int, default=1)
    gg.add_argument("--out", default="graph.txt")
    gg.add_argument("--weighted", action="store_true")
    gg.add_argument("--weight-min", type=int, default=1)
    gg.add_argument("--weight-max", type=int, default=100)
    gg.add_argument("--rmat-a", type=float, default=0.57)
    gg.add_argument("--rmat-b", type=float, default=0.19)
    gg.add_argument("--rmat-c", type=float, default=0.19)
    gg.add_argument("--rmat-d", type=float, default=0.05)
    gg.add_argument("--counter", action="store_true",
                    help="counter-based device generator (any scale) instead of the reference stream")
    gg.add_argument("--keep", type=float, default=0.55, help="grid: edge keep probability")
    gg.add_argument("--undirected", action="store_true", help="--counter: write the undirected CSR")
    gg.add_argument("--device", type=int, default=0)
    a = ap.parse_args(argv)
    try:
        if a.cmd == "run":
            return cmd_run(a)
        if a.cmd == "check":
            return cmd_check(a)
        return cmd_gen(a)
    except GraphdslError as e:
        print(f"error: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
