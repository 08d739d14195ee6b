import os, sys, socket
R = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, R)
import numpy as np, torch
import torch.multiprocessing as mp

def worker(rank, world, port):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK="0")
    import torch.distributed as dist
    import paper_2401_02472_b200 as G
    from paper_2401_02472_b200 import distributed as D
    from oracle import Port
    D.init_from_env("gloo")
    p = Port(); n = 1 << 12
    u, v = p.gen_rmat_edges(n, 16 * n, 21)
    gd = p.build_from_edges(n, u, v, None, True)
    ex = D.DeviceExecutor(G.DeviceGraph.from_csr(gd))
    roff = ex.rev_offsets()
    print(rank, "roff equal", np.array_equal(roff, gd.rev_offsets), "ranges", D.pr_ranges(roff, world), flush=True)
    orig = ex.pr_round
    def pr_round(rnd, *a):
        orig(rnd, *a)
        print(rank, "round", rnd, "dang_in", float(a[3][0]), "partials", a[-1].tolist(), "slice sum", float(a[-2].sum()), flush=True)
    ex.pr_round = pr_round
    r, rounds = D.sharded_pr(ex, 0.85, 1e-9, 6)
    print(rank, "rounds", rounds, flush=True)
    dist.destroy_process_group()

if __name__ == "__main__":
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    ctx = mp.get_context("spawn")
    ps = [ctx.Process(target=worker, args=(r, 2, port)) for r in range(2)]
    [x.start() for x in ps]; [x.join() for x in ps]
