import sys, os
R = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, R); sys.path.insert(0, os.path.join(R, "tests"))
import numpy as np, torch
import paper_2401_02472_b200 as G
from paper_2401_02472_b200 import distributed as D
from oracle import Port
from test_distributed import OracleExecutor
p = Port()
n = 1 << 12
u, v = p.gen_rmat_edges(n, 16 * n, 21)
gd = p.build_from_edges(n, u, v, None, True)
ranges = D.pr_ranges(gd.rev_offsets, 2)
print("ranges", ranges)
for kind in ("dev", "oracle"):
    exs = [D.DeviceExecutor(G.DeviceGraph.from_csr(gd)) if kind == "dev" else OracleExecutor(gd) for _ in ranges]
    chunk = max(b - a for a, b in ranges)
    contrib = [torch.zeros(n, dtype=torch.float64), torch.zeros(n, dtype=torch.float64)]
    parts = []
    for ex, (a, b) in zip(exs, ranges):
        ex.pr_setup(a, b)
        s = torch.zeros(chunk, dtype=torch.float64); pt = torch.zeros(2, dtype=torch.float64)
        ex.pr_init(s, pt)
        contrib[0][a:b] = s[:b - a]; parts.append(pt)
    dang = torch.tensor([float(sum(pt[0] for pt in parts))], dtype=torch.float64)
    for r in range(30):
        parts = []
        for ex, (a, b) in zip(exs, ranges):
            s = torch.zeros(chunk, dtype=torch.float64); pt = torch.zeros(2, dtype=torch.float64)
            ex.pr_round(r, 0.85, 1e-9, 110, dang, contrib[r & 1], s, pt)
            contrib[(r + 1) & 1][a:b] = s[:b - a]; parts.append(pt)
        dang = torch.tensor([float(sum(pt[0] for pt in parts))], dtype=torch.float64)
        uns = [float(pt[1]) for pt in parts]
        if r < 14 or r % 5 == 0:
            print(kind, r, "dang", float(dang[0]), "unsettled", uns, "csum", float(contrib[(r + 1) & 1].sum()))
        if sum(uns) == 0:
            print(kind, "rounds", r + 1); break
