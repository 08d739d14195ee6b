import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))), "tests"))
import numpy as np, torch
import paper_2401_02472_b200 as G
from oracle import Port
from test_distributed import OracleExecutor
p = Port()
n = 1 << 12
u, v = p.gen_rmat_edges(n, 16 * n, 21)
gd = p.build_from_edges(n, u, v, None, True)
dg = G.DeviceGraph.from_csr(gd)
for (a, b) in [(0, n), (0, 1500), (1500, n), (1501, n), (7, 3001)]:
    dg.pr_shard_setup(a, b)
    ox = OracleExecutor(gd); ox.pr_setup(a, b)
    cnt = b - a
    s_dev = torch.zeros(cnt, dtype=torch.float64, device="cuda"); part = torch.zeros(2, dtype=torch.float64, device="cuda")
    dg.pr_shard_init(s_dev, part)
    s_cpu = torch.zeros(cnt, dtype=torch.float64); part_c = torch.zeros(2, dtype=torch.float64)
    ox.pr_init(s_cpu, part_c)
    print((a, b), "init slice maxdiff", float((s_dev.cpu() - s_cpu).abs().max()), part.cpu().tolist(), part_c.tolist())
    rng = np.random.default_rng(0)
    contrib = torch.from_numpy(rng.random(n) * 1e-3)
    dang = torch.tensor([0.1], dtype=torch.float64)
    dg.pr_shard_round(0, 0.85, 1e-9, 110, dang.cuda(), contrib.cuda(), s_dev, part)
    ox.pr_round(0, 0.85, 1e-9, 110, dang, contrib, s_cpu, part_c)
    d = (s_dev.cpu() - s_cpu).abs() / s_cpu.abs().clamp(min=1e-300)
    bad = torch.nonzero(d > 1e-12).flatten()
    print("   round0 slice max rel", float(d.max()), "bad", bad[:10].tolist(), part.cpu().tolist(), part_c.tolist())
    r_dev = torch.zeros(cnt, dtype=torch.float64, device="cuda"); dg.pr_shard_rank(1, r_dev)
    r_c = torch.zeros(cnt, dtype=torch.float64); ox.pr_rank(1, r_c)
    print("   rank maxdiff", float((r_dev.cpu() - r_c).abs().max()))
