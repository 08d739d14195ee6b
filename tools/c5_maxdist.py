import sys, numpy as np
sys.path.insert(0, '/root/repo')
import paper_2401_02472_b200 as gdx
dg = gdx.DeviceGraph.generate("rmat", 1 << 26, 1 << 30, seed=1, directed=False, weights=(1, 100))
d = dg.sssp(0)
r = d[d < (2**63 - 1) // 2]
print("C5 reached", r.size, "max dist", r.max(), "quantiles", np.quantile(r, [0.5, 0.99, 0.9999]))
