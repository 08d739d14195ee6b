#!/usr/bin/env python3
"""Per-phase device time of the sharded SSSP loop (distributed.sharded_sssp) at
world size 1 over NCCL on C5 (or --scale), next to the single-GPU gdx_sssp.

  python tools/shard_probe.py [--scale 26] [--steps 2]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=26)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--rounds", action="store_true", help="print every round")
    a = ap.parse_args()
    import torch
    import torch.distributed as dist

    import paper_2401_02472_b200 as gdx
    from paper_2401_02472_b200 import distributed as D
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    os.environ.setdefault("RANK", "0")
    os.environ.setdefault("WORLD_SIZE", "1")
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
    sc = a.scale
    dg = gdx.DeviceGraph.generate("rmat", 1 << sc, 16 << sc, seed=1, directed=False,
                                  weights=(1, 100))
    ex = D.DeviceExecutor(dg)
    ex.offsets()
    for _ in range(a.steps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        st = {}
        D.sharded_sssp(ex, 0, to_host=False, stats=st)
        torch.cuda.synchronize()
        print(f"sharded_sssp: {(time.perf_counter() - t0) * 1e3:.1f} ms wall, {st}", flush=True)
    # phase breakdown (the loop of sharded_sssp with events)
    n = dg.n
    ex.sssp_setup(0, n)
    inf = (2**63 - 1) // 2
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    tot = {}
    for name, dt in (("int64", torch.int64),) + ((("int32", torch.int32),)
                                                  if hasattr(dg, "sssp_shard_frontier32") else ()):
        d = torch.full((n,), inf if dt == torch.int64 else 2**31 - 1, dtype=dt, device="cuda")
        prev = d.clone()
        d[0] = 0
        cnt = torch.zeros(2, dtype=torch.int64, device="cuda")
        torch.cuda.synchronize()
        t_start = time.perf_counter()
        ph = {"frontier": 0.0, "count_allreduce": 0.0, "relax": 0.0, "dist_allreduce": 0.0}
        rounds = 0
        while True:
            e = [ev() for _ in range(5)]
            e[0].record()
            if dt == torch.int64:
                c = ex.sssp_frontier(d, prev)
                o = 0
            else:
                c, o = ex.sssp_frontier32(d, prev)
            e[1].record()
            cnt[0], cnt[1] = c, o
            dist.all_reduce(cnt)
            done = int(cnt[0].item()) == 0
            e[2].record()
            if done:
                torch.cuda.synchronize()
                ph["frontier"] += e[0].elapsed_time(e[1])
                ph["count_allreduce"] += e[1].elapsed_time(e[2])
                break
            if dt == torch.int64:
                ex.sssp_relax(d)
            else:
                ex.sssp_relax32(d)
            e[3].record()
            dist.all_reduce(d, op=dist.ReduceOp.MIN)
            e[4].record()
            torch.cuda.synchronize()
            rounds += 1
            if a.rounds:
                print(f"  round {rounds}: items {c} frontier {e[0].elapsed_time(e[1]):.3f} ms "
                      f"relax {e[2].elapsed_time(e[3]):.3f} ms", flush=True)
            for k, (i, j) in zip(ph, ((0, 1), (1, 2), (2, 3), (3, 4))):
                ph[k] += e[i].elapsed_time(e[j])
        wall = (time.perf_counter() - t_start) * 1e3
        tot[name] = ph
        print(f"{name}: rounds {rounds} wall {wall:.1f} ms; " +
              ", ".join(f"{k} {v:.2f} ms" for k, v in ph.items()), flush=True)
    for _ in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        dg.sssp(0, out=torch.empty(n, dtype=torch.int64, device="cuda"))
        torch.cuda.synchronize()
        print(f"single-GPU gdx_sssp: {(time.perf_counter() - t0) * 1e3:.1f} ms wall", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
