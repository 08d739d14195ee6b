"""CPU: the CLI's value formatting matches interp::formatValue (std::to_chars)
and argument parsing; GPU: edge-list round trip and `run` end to end."""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT

from paper_2401_02472_b200.__main__ import format_value

VALUES = [0.5, 100.0, 1e-05, 0.0001, 0.001, 1e16, 1e22, 123456789.0, 1234.5, 0.1, 1.0 / 3.0,
          2.0 / 3.0 * 1e-7, 6.02e23, 1.7976931348623157e308, 5e-324, 0.15, 1e-4 * 3, 12345678901234567.0,
          2.5e-10, 3.0, 0.85, 1.0 / 262144.0]


@pytest.mark.skipif(shutil.which("g++") is None, reason="needs g++")
def test_format_value_matches_to_chars(tmp_path):
    src = tmp_path / "tc.cpp"
    src.write_text('#include <charconv>\n#include <cstdio>\n#include <cstdlib>\n'
                   'int main(int c, char** v) { for (int i = 1; i < c; ++i) { char b[64];'
                   ' double x = std::strtod(v[i], nullptr); auto r = std::to_chars(b, b + 64, x);'
                   ' *r.ptr = 0; std::printf("%s\\n", b); } }\n')
    exe = tmp_path / "tc"
    subprocess.run(["g++", "-std=c++17", "-O1", str(src), "-o", str(exe)], check=True)
    vals = VALUES + [-v for v in VALUES[:5]]
    out = subprocess.run([str(exe)] + [repr(v) for v in vals], capture_output=True, text=True,
                         check=True).stdout.split()
    assert [format_value(v) for v in vals] == out
    assert format_value(3) == "3" and format_value(True) == "true" and format_value(np.int64(-7)) == "-7"


def test_cli_parses_args():
    from paper_2401_02472_b200.__main__ import parse_args_kv
    a = parse_args_kv(["src=3", "sourceSet=0,1,5", "damping=0.85", "maxIter=7"], "x")
    assert a == {"src": 3, "sourceSet": [0, 1, 5], "damping": 0.85, "maxIter": 7}


@pytest.mark.gpu
def test_edge_list_round_trip_and_run(tmp_path, port):
    import paper_2401_02472_b200 as gdx
    p = tmp_path / "g.txt"
    p.write_text("# comment line\n0 1 5\n1 2 1\n\n0 2 7\n")  # test_csr.cpp:190-206
    g = gdx.DeviceGraph.load_edge_list(str(p), directed=False)
    h = g.download()
    assert (g.n, g.m) == (3, 6) and list(h.weights[:1]) == [5]
    p.write_text("0 oops\n")
    with pytest.raises(gdx.GraphdslError) as e:
        gdx.DeviceGraph.load_edge_list(str(p), directed=True)
    assert e.value.kind == "ParseError" and "malformed edge line" in str(e.value)
    # write -> load reproduces the graph
    u, v = port.gen_rmat_edges(500, 3000, 4)
    g = gdx.DeviceGraph.build_from_edges(500, u, v, None, False)
    g.set_hash_weights(1, 9, 3)
    out = tmp_path / "w.txt"
    g.write_edge_list(str(out), with_weights=True)
    g2 = gdx.DeviceGraph.load_edge_list(str(out), directed=False, node_count=500)
    a, b = g.download(), g2.download()
    for k in ("offsets", "dests", "weights"):
        assert np.array_equal(getattr(a, k), getattr(b, k)), k
    r = subprocess.run([sys.executable, "-m", "paper_2401_02472_b200", "run", "tc.sp", "--graph",
                        str(out)], capture_output=True, text=True, cwd=ROOT, timeout=300)
    assert r.returncode == 0, r.stderr
    assert r.stdout.strip().splitlines()[-1] == f"return\t{g.tc()}"


def _cli(*args, timeout=600):
    return subprocess.run([sys.executable, "-m", "paper_2401_02472_b200", *map(str, args)],
                          capture_output=True, text=True, cwd=ROOT, timeout=timeout)


@pytest.mark.gpu
@pytest.mark.parametrize("kind,weighted", [("rmat", True), ("uniform", False)])
def test_gen_graph_byte_identical_to_reference(tmp_path, ref, kind, weighted):
    """gen-graph writes the reference's file and summary line
    (graphdsl.cpp:265-296; restated over the reference library by the shim)."""
    ours, theirs = tmp_path / "ours.txt", tmp_path / "ref.txt"
    extra = ["--weighted", "--weight-min", "3", "--weight-max", "40"] if weighted else []
    r = _cli("gen-graph", "--kind", kind, "--nodes", 700, "--edges", 5000, "--seed", 11, "--out",
             ours, *extra)
    assert r.returncode == 0, r.stderr
    summary = ref.gen_graph_file(kind, 700, 5000, 11, theirs, weighted, 3, 40)
    assert ours.read_bytes() == theirs.read_bytes()
    assert r.stdout == summary.replace(str(theirs), str(ours))


@pytest.mark.gpu
def test_run_weight_options_match_with_random_weights(tmp_path, port):
    """run --weight-min/--weight-max/--weight-seed = CsrGraph::withRandomWeights
    (graphdsl.cpp:148-149, csr.cpp:172-195): the distances of the reweighted graph."""
    p = tmp_path / "g.txt"
    assert _cli("gen-graph", "--kind", "rmat", "--nodes", 512, "--edges", 4096, "--out",
                p).returncode == 0
    r = _cli("run", "sssp.sp", "--graph", p, "--arg", "src=3", "--weight-min", 1, "--weight-max",
             50, "--weight-seed", 9)
    assert r.returncode == 0, r.stderr
    import paper_2401_02472_b200 as gdx
    g = gdx.DeviceGraph.load_edge_list(str(p), directed=False)
    h = g.download()
    from conftest import G
    exp = port.sssp(port.with_random_weights(G(h.n, h.m, False, h.offsets, h.dests), 1, 50, 9), 3)
    got = [int(x.split("\t")[2]) for x in r.stdout.splitlines() if x.startswith("dist\t")]
    assert got == list(exp)


@pytest.mark.gpu
@pytest.mark.parametrize("prog,args", [("sssp.sp", ["--arg", "src=2"]), ("tc.sp", []),
                                       ("pr.sp", []), ("bc.sp", ["--arg", "sourceSet=0,5,9"])])
def test_check_passes(tmp_path, prog, args):
    """check: device fast path vs the textbook kernels, PASS at the corpus
    tolerance (graphdsl.cpp:175-256)."""
    p = tmp_path / "g.txt"
    assert _cli("gen-graph", "--kind", "rmat", "--nodes", 600, "--edges", 5000, "--weighted",
                "--out", p).returncode == 0
    directed = ["--directed"] if prog == "pr.sp" else []
    r = _cli("check", prog, "--graph", p, *directed, *args)
    assert r.returncode == 0, r.stdout + r.stderr
    lines = r.stdout.splitlines()
    assert lines[-1].startswith("PASS (tolerance ")
    if prog in ("sssp.sp", "tc.sp"):
        assert lines[-1] == "PASS (tolerance exact)"
        assert lines[0] == "sssp: max absolute distance error 0" if prog == "sssp.sp" else \
            lines[0].split()[2] == lines[0].split()[4]


@pytest.mark.gpu
def test_textbook_kernels_match_oracle(gdx, port):
    n = 1 << 11
    u, v = port.gen_rmat_edges(n, 16 * n, 12)
    und = port.with_random_weights(port.build_from_edges(n, u, v, None, False), 1, 100, 12)
    dr = port.build_from_edges(n, u, v, None, True)
    g, d = gdx.DeviceGraph.from_csr(und), gdx.DeviceGraph.from_csr(dr)
    assert np.array_equal(g.textbook_sssp(5), port.sssp(und, 5))
    assert g.textbook_tc() == port.tc(und) == g.tc()
    from conftest import rel_err
    assert rel_err(g.textbook_bc([0, 1, 2]), port.bc(und, [0, 1, 2])) < 1e-12
    r = d.textbook_pr(0.85, 1e-9, 110)
    e, _ = port.pr(dr, 0.85, 1e-9, 110)
    assert np.max(np.abs(r - e)) < 1e-6


GOLDEN_DIR = os.path.join(ROOT, "oracle", "_ref")


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(os.path.join(GOLDEN_DIR, "golden_tc")),
                    reason="golden units not built (make -C oracle golden-units)")
def test_units_match_golden_units(tmp_path):
    """bin/*_b200 keep the emitted units' command line and output
    (codegen_runtime.cpp:174-296): byte-identical to the reference's own
    generated CUDA units for SSSP and TC, within 1e-9 for PR and BC."""
    p = tmp_path / "g.txt"
    assert _cli("gen-graph", "--kind", "rmat", "--nodes", 900, "--edges", 7000, "--weighted",
                "--out", p).returncode == 0
    bins = os.path.join(ROOT, "paper_2401_02472_b200", "bin")
    cases = [("sssp", ["1", "4"]), ("tc", ["0"]), ("pr", ["1", "0.85", "1e-9", "110"]),
             ("bc", ["0", "0,3,7,11"])]
    for algo, args in cases:
        a = subprocess.run([os.path.join(bins, f"{algo}_b200"), str(p), *args],
                           capture_output=True, text=True, timeout=300)
        b = subprocess.run([os.path.join(GOLDEN_DIR, f"golden_{algo}"), str(p), *args],
                           capture_output=True, text=True, timeout=300)
        assert a.returncode == 0 == b.returncode, (algo, a.stderr, b.stderr)
        if algo in ("sssp", "tc"):
            assert a.stdout == b.stdout, algo
        else:
            la, lb = a.stdout.splitlines(), b.stdout.splitlines()
            assert len(la) == len(lb) and all(x.split("\t")[:2] == y.split("\t")[:2]
                                              for x, y in zip(la, lb))
            va = np.array([float(x.split("\t")[2]) for x in la])
            vb = np.array([float(y.split("\t")[2]) for y in lb])
            from conftest import rel_err
            assert rel_err(va, vb) < 1e-9, algo
    usage = subprocess.run([os.path.join(bins, "tc_b200")], capture_output=True, text=True)
    assert usage.returncode == 2 and "usage:" in usage.stderr
