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
