#!/usr/bin/env python3
"""C5 sharded SSSP at world 1 (NCCL) timed like bench.py (L2 flush, CUDA events
around the call) with the library profiler off and on."""
import os
import socket
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import torch.distributed as dist

    import paper_2401_02472_b200 as gdx
    from paper_2401_02472_b200 import distributed as D
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(sk.getsockname()[1]), RANK="0",
                      WORLD_SIZE="1", LOCAL_RANK="0")
    sk.close()
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
    dg = gdx.DeviceGraph.generate("rmat", 1 << 26, 1 << 30, seed=1, directed=False,
                                  weights=(1, 100))
    ex = D.DeviceExecutor(dg)
    ex.offsets()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    for prof in (False, True, False):
        dg.profile(prof)
        D.sharded_sssp(ex, 0, to_host=False)
        for _ in range(3):
            flush.fill_(1)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            a.record()
            st = {}
            D.sharded_sssp(ex, 0, to_host=False, stats=st)
            b.record()
            torch.cuda.synchronize()
            print(f"profile={prof}: events {a.elapsed_time(b):.1f} ms, wall "
                  f"{(time.perf_counter() - t0) * 1e3:.1f} ms, {st}", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
