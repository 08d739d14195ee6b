import os, sys, time
sys.path.insert(0, "/root/repo")
import paper_2401_02472_b200 as gdx
os.environ["GDX_SSSP_MODE"] = "scan"
dg = gdx.DeviceGraph.generate("rmat", 1 << 26, 1 << 30, seed=1, directed=False, weights=(1, 100))
dg.sssp(0)
dg.profile(True)
for i in range(2):
    dg.profile_reset()
    st = {}
    dg.sssp(0, stats=st)
    print(st["rounds"], dg.profile_read())
