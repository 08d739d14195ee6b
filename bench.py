#!/usr/bin/env python3
"""bench.py -- GTEPS of the B200 backend on the BASELINE.json configurations.

Headline (the `value` of the JSON line): config 2 of BASELINE.json --
PageRank pull (d=0.85, tol 1e-6, maxIter 100) on an RMAT scale-24 graph
(2^28 edge draws, ~263M directed edges), one gdx_pagerank call per step, graph
resident in HBM.  The other configs are reported under "per_algorithm":
C1 SSSP on the reference's own RMAT-18 graph and weights, C3 TC uniform 2^24,
C4 BC 64 sources on a 4899^2 grid, C5 SSSP RMAT-26 with ~2.1e9 stored edges.

Every config is checked after its timed region against the oracle on the same
graph ("parity": C1/C5 exact distances -- C1 also against the reference's own
interp::run, C5 also by an on-device certificate --, C2 ranks <= 1e-6 relative
with the same round count, C3 exact count, C4 all 64 sources <= 1e-6) and
carries a CPU baseline timed on the host's cores ("cpu_baseline").

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--algos sssp,tc,bc,sssp26] [--no-cpu-baseline] [--no-c5-cpu]

`--gpus N` > 1 runs one rank per GPU (self-launched through torch.distributed.run
when WORLD_SIZE is unset; fails if fewer than N GPUs are visible): PageRank
(headline), TC, BC and C5 SSSP run partitioned across the ranks (distributed.py;
strong scaling -- the graph is fixed), timing is the max over ranks.
`--impl reference` times the reference's own CPU path (oracle/_ref:
interp::run(ComputePR) in parallel mode on all host cores) on the same C2 graph,
one fixedPoint round per step.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "GTEPS per algorithm (SSSP/PR/TC/BC) at 1/2/4/8 B200; % of HBM roofline"
FLUSH_BYTES = 512 << 20  # > 126 MB L2


# ----------------------------------------------------------------------------- utils

def peaks() -> dict:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured (MEASURED_PEAKS.json)"}
    except Exception:
        return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


def ncu_summary() -> dict:
    """The committed ncu figures (profiles/ncu_summary.json)."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(p) as f:
            return json.load(f)
    except Exception:
        return {}


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], 0, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        try:
            for line in open(self.path):
                parts = [x.strip() for x in line.split(",")]
                if len(parts) < 9:
                    continue
                sm.append(float(parts[1]))
                mx = max(mx, float(parts[2]))
                for nm, val in zip(names, parts[5:9]):
                    if val.lower().startswith("active"):
                        reasons.add(nm)
            os.unlink(self.path)
        except Exception:
            pass
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "samples": len(sm), "reasons": sorted(reasons)}


class Dist:
    def __init__(self):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.pg = None

    def init(self, torch, force: bool = False):
        torch.cuda.set_device(self.local)
        if self.world > 1 or force:
            import torch.distributed as dist
            if "RANK" not in os.environ:  # --sharded without torchrun: a 1-rank group
                import socket
                sk = socket.socket()
                sk.bind(("127.0.0.1", 0))
                os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(sk.getsockname()[1]),
                                  RANK="0", WORLD_SIZE="1", LOCAL_RANK="0")
                sk.close()
            dist.init_process_group("nccl", device_id=torch.device("cuda", self.local))
            self.pg = dist

    def barrier(self, torch):
        if self.pg:
            self.pg.barrier()
        torch.cuda.synchronize()

    def max(self, torch, x: float) -> float:
        if not self.pg:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        self.pg.all_reduce(t, op=self.pg.ReduceOp.MAX)
        return float(t.item())

    def close(self):
        if self.pg:
            self.pg.destroy_process_group()


# ------------------------------------------------------------------------ our arm

def timed_steps(torch, dist, step, steps: int, warmup: int, flush, keep_all: bool = True):
    """W warm-up steps, then K steps each preceded by an L2 flush; returns
    (per-step ms list, bracketed total ms).  Device time via CUDA events on the
    current stream (the library runs on it, see gdx_graph_set_stream)."""
    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(steps)]
    # keep_all=False keeps only the last step's result: holding every step's
    # device output (C5's 537 MB distance vector) would make the later steps
    # allocate under memory pressure inside the timed region
    results = []
    dist.barrier(torch)
    t0 = time.perf_counter()
    for a, b in evs:
        flush.zero_()
        if not keep_all:
            results = []  # the previous step's output freed before this step allocates its own
        a.record()
        r = step()
        results = results + [r] if keep_all else [r]
        del r
        b.record()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) * 1e3
    dist.barrier(torch)
    return [a.elapsed_time(b) for a, b in evs], wall, results


def roofline(prof: dict, kernel: str, algo_bytes: float, pk: dict, work_launches=None,
             traffic_key=None) -> dict:
    """achieved = algorithmic bytes / summed device time of `kernel` (CUDA events
    around every launch, recorded by the library on the launching stream).
    `kernel` may be "a+b": kernels that together make one unit of work (a PR
    round, an SSSP call), timed and counted together.  `work_launches` = the
    number of units (PR: rounds that did work; others: calls).  traffic = DRAM
    bytes per unit from the committed ncu captures (profiles/ncu_summary.json:
    `traffic_key` -> dram_bytes_per_unit, else the per-kernel launch figures)."""
    parts = kernel.split("+")
    ms = sum(prof.get(k, (0.0, 0))[0] for k in parts)
    launches = prof.get(parts[0], (0.0, 0))[1]
    if work_launches:
        launches = work_launches
    achieved = algo_bytes / (ms * 1e-3) / 1e9 if ms > 0 else 0.0
    traffic, known = None, []
    summ = ncu_summary()
    if traffic_key and traffic_key in summ and "dram_bytes_per_unit" in summ[traffic_key]:
        traffic, known = summ[traffic_key]["dram_bytes_per_unit"], [traffic_key]
    else:
        tr = {k: summ.get(k, {}).get("dram_bytes_per_launch") for k in parts}
        known = [k for k, t in tr.items() if t is not None]
        traffic = sum(tr[k] for k in known) if known else None
    return {"kernel": kernel, "bound": "hbm", "achieved": round(achieved, 1),
            "peak": pk["hbm_gbs"], "unit": "GB/s", "frac": round(achieved / pk["hbm_gbs"], 4),
            "peak_source": pk["source"], "traffic": traffic, "traffic_source": known,
            "kernel_ms_per_unit": round(ms / max(launches, 1), 4), "units": launches,
            "algorithmic_bytes_per_unit": round(algo_bytes / max(launches, 1), 1)}


# ------------------------------------------------------------------ parity + CPU legs
# The oracle (oracle/, test infrastructure) is the checker here and the CPU
# baseline: it runs after a config's timed region, on the same graph, and is
# never the thing measured.

CORES = os.cpu_count() or 1


def _port():
    from oracle import Port
    return Port()


def _ref():
    from oracle import Ref, ref_available
    return Ref() if ref_available() else None


def rel_err(a, b) -> float:
    import numpy as np
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    if a.size == 0:
        return 0.0
    scale = np.maximum(np.maximum(np.abs(a), np.abs(b)), 1e-12)
    return float(np.max(np.abs(a - b) / scale))


def timed_cpu(fn, budget_s: float):
    """Whole runs of fn() until >= budget_s; returns (last result, runs, seconds)."""
    runs, t0, res = 0, time.perf_counter(), None
    while True:
        res = fn()
        runs += 1
        t = time.perf_counter() - t0
        if t >= budget_s:
            return res, runs, t


def _to_host(x):
    import numpy as np
    return x.cpu().numpy() if hasattr(x, "cpu") else np.asarray(x)


# ------------------------------------------------------------------------ our arm

def bench_pr(torch, gdx, dist, args, pk, cpu_legs: bool) -> dict:
    scale, draws = 24, 1 << 28
    dg = gdx.DeviceGraph.generate("rmat", 1 << scale, draws, seed=1, directed=True,
                                  device=dist.local)
    n, m = dg.n, dg.m
    dg.set_stream(torch.cuda.current_stream().cuda_stream)
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    flush = torch.empty(FLUSH_BYTES, dtype=torch.uint8, device="cuda")
    stats = {}

    def step():
        _, rounds = dg.pagerank(0.85, 1e-6, 100, out=out, stats=stats)
        return rounds

    dg.profile(True)
    for _ in range(args.warmup):
        step()
    warm = dg.profile_read()  # the renumbering (csrc/relabel.cu) is built in the warm-up
    dg.profile_reset()
    with Clocks(dist.local) as clk:
        ms, wall, rounds = timed_steps(torch, dist, step, args.steps, 0, flush)
    prof = dg.profile_read()
    dg.profile(False)
    total_ms = dist.max(torch, sum(ms))
    edges = float(m) * sum(rounds)
    res = {
        "workload": "C2 PageRank pull RMAT-24 (2^28 draws, directed) d=0.85 tol=1e-6 maxIter=100",
        "n": n, "m": m, "rounds": rounds[-1], "gteps": edges * dist.world / (total_ms * 1e-3) / 1e9,
        "ms_per_step": total_ms / args.steps, "wall_ms": wall,
        "roofline": roofline(prof, "pr_edges+pr_cross+pr_vertices", sum(rounds) * (12.0 * m + 24.0 * n), pk,
                             work_launches=sum(rounds), traffic_key="pr_round"),
        "clocks": clk.summary(), "gpu_launches": int(sum(v[1] for v in prof.values())),
        "kernels": {k: {"ms": round(v[0], 3), "launches": v[1]} for k, v in prof.items()},
    }
    res["roofline"]["bytes_formula"] = "per round 12 m + 24 n (SURVEY.md 8(d))"
    if "relabel" in warm:
        res["renumbering"] = {"build_ms": round(warm["relabel"][0], 3), "note": (
            "degree-ordered renumbering (csrc/relabel.cu) built by the handle's second call "
            "(warm-up) and kept; the timed calls run on it, the e2e leg (one call per upload) "
            "does not")}
    ranks = _to_host(out)
    # ---- e2e: host CSR arrays -> C ABI (upload) -> PR -> host rank --------------
    h = dg.download(("offsets", "rev_offsets", "rev_srcs"))
    pin = {k: torch.from_numpy(getattr(h, k)).pin_memory() for k in ("offsets", "rev_offsets", "rev_srcs")}
    rank_host = torch.empty(n, dtype=torch.float64).pin_memory()

    class View:
        pass

    v = View()
    v.n, v.m, v.directed = n, m, True
    v.offsets, v.rev_offsets, v.rev_srcs = pin["offsets"], pin["rev_offsets"], pin["rev_srcs"]
    v.dests = v.weights = v.rev_eid = None

    def e2e_step():
        g2 = gdx.DeviceGraph.from_csr(v, device=dist.local)
        _, r = g2.pagerank(0.85, 1e-6, 100, out=rank_host)
        g2.close()
        return r

    dg.close()
    for _ in range(args.warmup):
        e2e_step()
    dist.barrier(torch)
    t0 = time.perf_counter()
    rr = []
    for _ in range(args.steps):
        rr.append(e2e_step())
    e2e_s = dist.max(torch, time.perf_counter() - t0)
    res["e2e"] = {"value": float(m) * sum(rr) * dist.world / e2e_s / 1e9, "unit": "GTEPS",
                  "h2d_bytes_per_step": int(sum(t.numel() * 4 for t in pin.values())),
                  "d2h_bytes_per_step": int(n * 8), "ms_per_step": e2e_s * 1e3 / args.steps,
                  "path": "gdx_graph_create(host CSR) + gdx_pagerank(host out) + destroy"}
    if cpu_legs:
        port = _port()

        class HG:  # the port reads the reverse CSR for the gather
            pass
        hg = HG()
        hg.n, hg.m, hg.directed = n, m, True
        hg.offsets, hg.rev_offsets, hg.rev_srcs = h.offsets, h.rev_offsets, h.rev_srcs
        hg.dests = hg.weights = hg.rev_eid = None
        (ranks_cpu, r_cpu), runs, t = timed_cpu(
            lambda: port.pr(hg, 0.85, 1e-6, 100, threads=CORES), args.cpu_budget)
        res["cpu_baseline"] = {
            "value": float(m) * r_cpu * runs / t / 1e9, "unit": "GTEPS", "cores": CORES,
            "kind": "port",
            "sample": f"oracle port (oracle/gdx_oracle.cpp orc_pr: ComputePR d=0.85 tol=1e-6 "
                      f"maxIter=100, per-node ascending gathers) on the same C2 graph, {runs} "
                      f"full runs x {r_cpu} rounds on {CORES} threads in {t:.1f}s"}
        err = rel_err(ranks, ranks_cpu)
        # the e2e leg's ranks too: a freshly uploaded graph's first call runs on
        # the caller's numbering, the timed calls on the renumbered handle
        err_e2e = rel_err(rank_host.numpy(), ranks_cpu)
        res["parity"] = {"ok": bool(max(err, err_e2e) <= 1e-6 and r_cpu == rounds[-1] == rr[-1]),
                         "vs": "oracle port pr", "max_rel_err": err, "e2e_max_rel_err": err_e2e,
                         "tolerance": "1e-6 relative per node",
                         "rounds": rounds[-1], "rounds_e2e": rr[-1], "rounds_oracle": r_cpu}
    return res


def sssp_certificate(torch, dg, d) -> bool:
    """Size-independent SSSP check on the device: d[src]=0, every edge
    satisfies d[v] <= d[u] + w, every other reached vertex has a tight in-edge
    (so d is the unique shortest-path distance vector)."""
    INF = (2**63 - 1) // 2
    off, dst, w = dg.device_arrays(["offsets", "dests", "weights"])
    offl = off.long()
    tight = torch.zeros(dg.n, dtype=torch.bool, device=d.device)
    ok = True
    chunk = 1 << 27
    for e0 in range(0, dg.m, chunk):
        e1 = min(dg.m, e0 + chunk)
        eid = torch.arange(e0, e1, device=d.device, dtype=torch.int64)
        src = torch.searchsorted(offl, eid, right=True) - 1
        du, dv = d[src], d[dst[e0:e1].long()]
        fin = du < INF
        cand = du + w[e0:e1].long()
        ok &= bool(torch.all(~fin | (dv <= cand)))
        tight.index_fill_(0, dst[e0:e1].long()[fin & (dv == cand)], True)
        del eid, src, du, dv, fin, cand
    reached = d < INF
    ok &= int(d[0]) == 0
    tight[0] = True
    ok &= bool(torch.all(~reached | tight))
    del off, dst, w, offl, tight
    return ok


def sssp_roofline(prof, sts, pk, n, traffic_key):
    kern = ("sssp_graph" if "sssp_graph" in prof else
            "sssp_relax+sssp_frontier" if "sssp_relax" in prof else "sssp_rounds")
    r = roofline(prof, kern, sum(s["algorithmic_bytes"] for s in sts), pk,
                 traffic_key=traffic_key, work_launches=len(sts))
    r["bytes_formula"] = "16 V_vis + 12 E_vis + 8 U (SURVEY.md 8(d))"
    s = sts[-1]
    r["counters_per_call"] = {"V_vis": s["vertices_visited"], "E_vis": s["edges_visited"],
                              "U": s["updates"], "rounds": s["rounds"]}
    # the frontier scan reads dist + prev for all n vertices per round (+ the
    # final empty round): work the formula does not count
    r["scan_bytes_per_call"] = float((s["rounds"] + 1) * 2 * 4 * n)
    return r


def bench_sssp(torch, gdx, dist, args, pk, scale: int, cpu_legs: bool) -> dict:
    if scale == 18:
        # C1 on the reference's own graph: genRmatEdges(2^18,
        # 2^22, 1) undirected, withRandomWeights(1, 100, 1) -- the reference's
        # mt19937_64 streams from libgdx's host side, the CSR built on the GPU
        u, v = gdx.gen_rmat_edges(1 << 18, 1 << 22, 1)
        dg = gdx.DeviceGraph.build_from_edges(1 << 18, u, v, None, directed=False,
                                              device=dist.local)
        dg.set_random_weights(1, 100, 1)
        cfg, recipe = "C1", ("genRmatEdges(2^18, 2^22, seed 1) undirected + withRandomWeights(1, "
                             "100, seed 1): the reference's own graph")
    else:
        dg = gdx.DeviceGraph.generate("rmat", 1 << scale, 16 << scale, seed=1, directed=False,
                                      weights=(1, 100), device=dist.local)
        cfg, recipe = "C5", (f"counter-based RMAT-{scale} twin, 2^{scale + 4} draws, undirected, "
                             "counter-hash weights U[1,100]")
    dg.set_stream(torch.cuda.current_stream().cuda_stream)
    out = torch.empty(dg.n, dtype=torch.int64, device="cuda")
    flush = torch.empty(FLUSH_BYTES, dtype=torch.uint8, device="cuda")
    st_all = []

    def step():
        st = {}
        dg.sssp(0, out=out, stats=st)
        st_all.append(st)
        return st

    dg.profile(True)
    for _ in range(args.warmup):
        step()
    warm = dg.profile_read()
    dg.profile_reset()
    st_all.clear()
    ms, wall, sts = timed_steps(torch, dist, step, args.steps, 0, flush)
    prof = dg.profile_read()
    total = dist.max(torch, sum(ms))
    res = {"workload": f"{cfg} SSSP RMAT-{scale} ef16 undirected, weights U[1,100], src 0",
           "graph": recipe, "n": dg.n, "m": dg.m, "rounds": sts[-1]["rounds"],
           "edges_visited_over_m": sts[-1]["edges_visited"] / dg.m,
           "gteps": dg.m * args.steps * dist.world / (total * 1e-3) / 1e9,
           "ms_per_step": total / args.steps,
           "roofline": sssp_roofline(prof, sts, pk, dg.n, f"sssp_{cfg.lower()}_call"),
           "gpu_launches": int(sum(s["launches"] for s in sts))}
    if "relabel" in warm:
        res["renumbering"] = {"build_ms": round(warm["relabel"][0], 3), "note": (
            "degree-ordered renumbering with rows sorted by the new ids (csrc/relabel.cu), "
            "built by the handle's second call (warm-up) and kept")}
    if scale > 18:
        res["certificate_ok"] = sssp_certificate(torch, dg, out)
    if cpu_legs:
        port = _port()
        d = _to_host(out)
        h = dg.download(("offsets", "dests", "weights"))
        dg.close()
        del out, flush
        torch.cuda.empty_cache()
        t0 = time.perf_counter()
        exp = port.sssp(h, 0)
        t_dij = time.perf_counter() - t0
        par = {"ok": bool((d == exp).all()), "vs": "oracle port sssp (Dijkstra, oracles.cpp:10-31)",
               "mismatches": int((d != exp).sum()), "tolerance": "exact int64"}
        if scale == 18:
            ref = _ref()
            if ref is not None:  # the reference itself: interp::run(ComputeSSSP), parallel
                rg = ref.build_from_host(h)
                (di, mod, fin), runs, t = timed_cpu(
                    lambda: rg.interp_sssp(0, parallel=True, threads=CORES), args.cpu_budget)
                par["interp_ok"] = bool((di == d).all() and not mod.any() and fin)
                par["ok"] = par["ok"] and par["interp_ok"]
                res["cpu_baseline"] = {
                    "value": dg_m(h) * runs / t / 1e9, "unit": "GTEPS", "cores": CORES,
                    "kind": "reference",
                    "sample": f"interp::run(ComputeSSSP, src 0) ExecMode::Parallel on {CORES} "
                              f"threads (oracle/_ref), same C1 graph, {runs} runs in {t:.1f}s"}
        if "cpu_baseline" not in res:
            res["cpu_baseline"] = {
                "value": dg_m(h) / t_dij / 1e9, "unit": "GTEPS", "cores": 1, "kind": "port",
                "sample": f"oracle port Dijkstra (oracles.cpp:10-31) on the same {cfg} graph, "
                          f"one full run in {t_dij:.1f}s"}
        res["parity"] = par
    else:
        dg.close()
    torch.cuda.empty_cache()
    return res


def dg_m(h) -> float:
    return float(h.m)


def bench_tc(torch, gdx, dist, args, pk, cpu_legs: bool) -> dict:
    dg = gdx.DeviceGraph.generate("uniform", 1 << 24, 1 << 27, seed=1, directed=False,
                                  device=dist.local)
    dg.set_stream(torch.cuda.current_stream().cuda_stream)
    flush = torch.empty(FLUSH_BYTES, dtype=torch.uint8, device="cuda")
    sts = []

    def step():
        st = {}
        c = dg.tc(stats=st)
        sts.append(st)
        return c

    dg.profile(True)
    t0 = time.perf_counter()
    step()  # first call on the handle: builds the oriented CSR (a cached plan)
    plan_ms = (time.perf_counter() - t0) * 1e3
    plan_prof = dg.profile_read()
    for _ in range(args.warmup):
        step()
    dg.profile_reset()
    sts.clear()
    ms, wall, counts = timed_steps(torch, dist, step, args.steps, 0, flush)
    prof = dg.profile_read()
    total = dist.max(torch, sum(ms))
    kern = "+".join(k for k in ("tc", "tc_heavy") if k in prof)
    res = {"workload": "C3 TC uniform 2^24 vertices, 2^27 draws, undirected",
           "n": dg.n, "m": dg.m, "triangles": counts[-1],
           "gteps": dg.m * args.steps * dist.world / (total * 1e-3) / 1e9,
           "ms_per_step": total / args.steps,
           "roofline": roofline(prof, kern, sum(s["algorithmic_bytes"] for s in sts), pk,
                                traffic_key="tc_call", work_launches=len(sts)),
           "plan": {"first_call_ms": round(plan_ms, 2),
                    "orientation_kernels_ms": round(sum(plan_prof.get(k, (0, 0))[0] for k in
                                                        ("tc_orient", "tc_orient_fill")), 3),
                    "signature_kernels_ms": round(plan_prof.get("tc_sig", (0, 0))[0], 3),
                    "note": "the oriented CSR (off+, adj+) and the pair-filter signatures "
                            "are built by the first call on a handle and cached with it, "
                            "like the PageRank plan"},
           "gpu_launches": int(sum(v[1] for v in prof.values())),
           "kernels": {k: {"ms": round(v[0], 3), "launches": v[1]} for k, v in prof.items()}}
    res["roofline"]["bytes_formula"] = ("4(n+1) + 4m + 4 * sum over oriented edges u->v of "
                                        "(d+(u) + d+(v)) (SURVEY.md 8(d))")
    if cpu_legs:
        port = _port()
        h = dg.download(("offsets", "dests"))
        dg.close()
        c_cpu, runs, t = timed_cpu(lambda: port.tc(h, threads=CORES), 0.0)
        res["cpu_baseline"] = {
            "value": float(h.m) * runs / t / 1e9, "unit": "GTEPS", "cores": CORES, "kind": "port",
            "sample": f"oracle port TC (tc.sp:6-18 semantics) on the same C3 graph, {runs} full "
                      f"run(s) on {CORES} threads in {t:.1f}s"}
        res["parity"] = {"ok": bool(c_cpu == counts[-1]), "vs": "oracle port tc",
                         "triangles_oracle": int(c_cpu), "tolerance": "exact int64"}
    else:
        dg.close()
    return res


def bench_bc(torch, gdx, dist, args, pk, cpu_legs: bool) -> dict:
    import numpy as np
    side = 4899
    dg = gdx.DeviceGraph.generate("grid", side, seed=1, keep=0.55, directed=False,
                                  device=dist.local)
    dg.set_stream(torch.cuda.current_stream().cuda_stream)
    h = dg.download(("offsets", "dests"))
    deg = np.diff(h.offsets)
    cand = np.flatnonzero(deg > 0)
    rng = np.random.default_rng(1)
    sources = sorted(rng.choice(cand, size=args.bc_sources, replace=False).tolist())
    out = torch.empty(dg.n, dtype=torch.float64, device="cuda")
    flush = torch.empty(FLUSH_BYTES, dtype=torch.uint8, device="cuda")
    sts = []

    def step():
        st = {}
        dg.bc(sources, out=out, stats=st)
        sts.append(st)
        return st

    dg.profile(True)
    for _ in range(args.warmup):
        step()
    dg.profile_reset()
    sts.clear()
    steps = max(1, args.steps // 2)
    ms, wall, _ = timed_steps(torch, dist, step, steps, 0, flush)
    prof = dg.profile_read()
    total = dist.max(torch, sum(ms))
    kern = "bc_cta" if "bc_cta" in prof else "bc_forward+bc_backward"
    res = {"workload": f"C4 BC {len(sources)} sources, {side}^2 grid keep 0.55 undirected",
           "n": dg.n, "m": dg.m, "levels": sts[-1]["rounds"], "steps": steps,
           "gteps": dg.m * len(sources) * steps * dist.world / (total * 1e-3) / 1e9,
           "ms_per_step": total / steps,
           "roofline": roofline(prof, kern, sum(s["algorithmic_bytes"] for s in sts), pk,
                                traffic_key="bc_call", work_launches=len(sts)),
           "gpu_launches": int(sum(v[1] for v in prof.values()))}
    s = sts[-1]
    res["roofline"]["bytes_formula"] = ("per source 48 n_reached + 16 m_scanned + 24 m_dag "
                                        "(SURVEY.md 8(d))")
    # summed over the call's sources: reached (s, v) pairs, edges the forward
    # pass scanned, DAG edges (each counted once)
    res["roofline"]["counters_per_call"] = {"n_reached": s["vertices_visited"],
                                            "m_scanned": s["edges_visited"],
                                            "m_dag": s["updates"]}
    if cpu_legs:
        port = _port()
        b = _to_host(out)
        dg.close()
        del out, flush
        torch.cuda.empty_cache()
        t0 = time.perf_counter()
        exp = port.bc(h, sources, threads=CORES)
        t = time.perf_counter() - t0
        err = rel_err(b, exp)
        res["cpu_baseline"] = {
            "value": float(h.m) * len(sources) / t / 1e9, "unit": "GTEPS", "cores": CORES,
            "kind": "port",
            "sample": f"oracle port Brandes (oracles.cpp:33-71, sources in parallel on {CORES} "
                      f"threads, summed in source order) on the same C4 graph and all "
                      f"{len(sources)} sources in {t:.1f}s"}
        res["parity"] = {"ok": bool(err <= 1e-6 and np.isfinite(b).all()), "vs": "oracle port bc",
                         "sources_compared": len(sources), "max_rel_err": err,
                         "tolerance": "1e-6 relative per node"}
    else:
        dg.close()
    return res


# --------------------------------------------------------------- sharded (N > 1) arm

def _shard_roofline(prof, kernels, algo_bytes, pk, launches):
    r = roofline(prof, kernels, algo_bytes, pk, work_launches=launches)
    r["scope"] = "rank 0's kernels and rank 0's share of the algorithmic bytes"
    return r


def bench_pr_sharded(torch, gdx, dist, args, pk) -> dict:
    """C2 PageRank partitioned over the ranks by destination-vertex ranges.
    The exchange is fused into the kernels over peer memory
    (distributed.sharded_pr_p2p); if that fails, per round one NCCL all-gather
    of the contrib slices and one all-reduce (distributed.sharded_pr).
    Strong scaling: the graph is fixed, every rank computes its rows."""
    from paper_2401_02472_b200 import distributed as D
    dg = gdx.DeviceGraph.generate("rmat", 1 << 24, 1 << 28, seed=1, directed=True,
                                  device=dist.local)
    n, m = dg.n, dg.m
    ex = D.DeviceExecutor(dg)
    flush = torch.empty(FLUSH_BYTES, dtype=torch.uint8, device="cuda")

    # exchange: fused into the kernels over peer memory (NVLink P2P through CUDA
    # IPC, gdx_pr_p2p_*); NCCL all-gather + all-reduce if peer memory fails
    exchange = {"kind": "p2p"}

    def step():
        if exchange["kind"] == "p2p":
            _, rounds = D.sharded_pr_p2p(ex, 0.85, 1e-6, 100, to_host=False)
        else:
            _, rounds = D.sharded_pr(ex, 0.85, 1e-6, 100, to_host=False)
        return rounds

    try:
        step()
    except Exception as e:  # noqa: BLE001 -- recorded in the JSON line
        exchange.update(kind="nccl", p2p_error=str(e)[:200])
    dg.profile(True)
    for _ in range(args.warmup):
        step()
    dg.profile_reset()
    with Clocks(dist.local) as clk:
        ms, wall, rounds = timed_steps(torch, dist, step, args.steps, 0, flush)
    prof = dg.profile_read()
    dg.profile(False)
    total_ms = dist.max(torch, sum(ms))
    # the partition the rounds ran on (the renumbered graph's, when
    # gdx_pagerank renumbers this one: distributed._renumbered)
    ren = D._renumbered(ex, "pr")
    pex = ren[0] if ren is not None else ex
    ranges = D.pr_ranges(pex.rev_offsets(), dist.world)
    roff = pex.rev_offsets()
    v0, v1 = ranges[dist.rank]
    e_r = int(roff[v1]) - int(roff[v0])
    res = {
        "workload": "C2 PageRank pull RMAT-24 (2^28 draws, directed) d=0.85 tol=1e-6 maxIter=100",
        "n": n, "m": m, "rounds": rounds[-1],
        "gteps": float(m) * sum(rounds) / (total_ms * 1e-3) / 1e9,
        "ms_per_step": total_ms / args.steps, "wall_ms": wall,
        "roofline": _shard_roofline(prof, "pr_edges+pr_cross+pr_vertices",
                                    sum(rounds) * (12.0 * e_r + 24.0 * (v1 - v0)), pk, sum(rounds)),
        "clocks": clk.summary(), "gpu_launches": int(sum(v[1] for v in prof.values())),
        "kernels": {k: {"ms": round(v[0], 3), "launches": v[1]} for k, v in prof.items()},
        "partition": {"ranges": ranges, "rank0_edges": e_r},
        "exchange": exchange,
    }
    # e2e: every rank uploads the host CSR through the C ABI, runs the sharded
    # fixedPoint and gathers the full rank vector to the host
    h = dg.download()
    pin = {k: torch.from_numpy(getattr(h, k)).pin_memory() for k in ("offsets", "rev_offsets", "rev_srcs")}

    class View:
        pass

    v = View()
    v.n, v.m, v.directed = n, m, True
    v.offsets, v.rev_offsets, v.rev_srcs = pin["offsets"], pin["rev_offsets"], pin["rev_srcs"]
    v.dests = v.weights = v.rev_eid = None

    rank_host = torch.empty(n, dtype=torch.float64).pin_memory()

    def e2e_step():
        # the same exchange as the timed rounds; the full rank vector lands in
        # pinned host memory
        g2 = gdx.DeviceGraph.from_csr(v, device=dist.local)
        ex2 = D.DeviceExecutor(g2)
        if exchange["kind"] == "p2p":
            out, r = D.sharded_pr_p2p(ex2, 0.85, 1e-6, 100, to_host=False)
        else:
            out, r = D.sharded_pr(ex2, 0.85, 1e-6, 100, to_host=False)
        rank_host.copy_(out)
        g2.close()
        return r

    dg.close()
    for _ in range(args.warmup):
        e2e_step()
    dist.barrier(torch)
    t0 = time.perf_counter()
    rr = [e2e_step() for _ in range(args.steps)]
    e2e_s = dist.max(torch, time.perf_counter() - t0)
    res["e2e"] = {"value": float(m) * sum(rr) / e2e_s / 1e9, "unit": "GTEPS",
                  "h2d_bytes_per_step": int(sum(t.numel() * 4 for t in pin.values())),
                  "d2h_bytes_per_step": int(n * 8), "ms_per_step": e2e_s * 1e3 / args.steps,
                  "path": f"per rank: gdx_graph_create(host CSR) + sharded PR ({exchange['kind']}) "
                          "+ rank gather to pinned host memory"}
    return res


def bench_sharded_other(torch, gdx, dist, args, pk, algo: str) -> dict:
    """C3 TC (owner-vertex ranges + one all-reduce), C4 BC (source blocks + one
    all-reduce of bc), C5 SSSP (vertex ranges, MIN all-reduce per round)."""
    import numpy as np
    from paper_2401_02472_b200 import distributed as D
    flush = torch.empty(FLUSH_BYTES, dtype=torch.uint8, device="cuda")
    if algo == "tc":
        dg = gdx.DeviceGraph.generate("uniform", 1 << 24, 1 << 27, seed=1, directed=False,
                                      device=dist.local)
        ex = D.DeviceExecutor(dg)
        ex.offsets()

        def step():
            return D.sharded_tc(ex)
        units, name, kern = float(dg.m), "C3 TC uniform 2^24 vertices, 2^27 draws, undirected", \
            "tc+tc_orient+tc_orient_fill"
    elif algo == "bc":
        side = 4899
        dg = gdx.DeviceGraph.generate("grid", side, seed=1, keep=0.55, directed=False,
                                      device=dist.local)
        ex = D.DeviceExecutor(dg)
        deg = np.diff(ex.offsets())
        rng = np.random.default_rng(1)
        sources = sorted(rng.choice(np.flatnonzero(deg > 0), size=args.bc_sources,
                                    replace=False).tolist())

        def step():
            return D.sharded_bc(ex, sources, to_host=False)
        units, name, kern = float(dg.m) * len(sources), \
            f"C4 BC {len(sources)} sources, {side}^2 grid keep 0.55 undirected", "bc_forward"
    else:  # sssp26
        dg = gdx.DeviceGraph.generate("rmat", 1 << 26, 1 << 30, seed=1, directed=False,
                                      weights=(1, 100), device=dist.local)
        ex = D.DeviceExecutor(dg)
        ex.offsets()
        st = {}
        # exchange fused into the relaxation over peer memory (gdx_sssp_p2p_*);
        # the NCCL rounds (distributed.sharded_sssp) if peer memory fails
        exchange = {"kind": "p2p"}
        try:
            D.sharded_sssp_p2p(ex, 0, to_host=False)
        except Exception as e:  # noqa: BLE001 -- recorded in the JSON line
            exchange.update(kind="nccl", p2p_error=str(e)[:200])

        def step():
            if exchange["kind"] == "p2p":
                return D.sharded_sssp_p2p(ex, 0, to_host=False, stats=st)
            return D.sharded_sssp(ex, 0, to_host=False, stats=st)
        units, name, kern = float(dg.m), \
            "C5 SSSP RMAT-26 ef16 undirected, weights U[1,100], src 0", "sssp_multi_graph"
    dg.profile(True)
    for _ in range(args.warmup):  # W >= 3 (the second C5 call still pays ~60 ms of first-use cost)
        step()
    dg.profile_reset()
    steps = max(1, args.steps // 2) if algo == "bc" else args.steps
    ms, wall, outs = timed_steps(torch, dist, step, steps, 0, flush, keep_all=False)
    if dist.rank == 0:
        print(f"{algo} sharded steps (ms): " + " ".join(f"{x:.1f}" for x in ms), file=sys.stderr)
    prof = dg.profile_read()
    total = dist.max(torch, sum(ms))
    res = {"workload": name, "n": dg.n, "m": dg.m, "steps": steps,
           "gteps": units * steps / (total * 1e-3) / 1e9, "ms_per_step": total / steps,
           "parallelism": f"sharded x{dist.world}", "scaling": "strong",
           "gpu_launches": int(sum(v[1] for v in prof.values())),
           "kernels": {k: {"ms": round(v[0], 3), "launches": v[1]} for k, v in prof.items()}}
    if algo == "tc":
        res["triangles"] = outs[-1]
    if algo == "sssp26":
        res["rounds"] = st.get("rounds")
        res["exchange"] = exchange
        res["certificate_ok"] = sssp_certificate(torch, dg, outs[-1])
    dg.close()
    torch.cuda.empty_cache()
    return res


def run_ours(args) -> None:
    import torch

    import paper_2401_02472_b200 as gdx
    dist = Dist()
    dist.init(torch, force=args.sharded)
    pk = peaks()
    algos = [a for a in args.algos.split(",") if a]
    cpu = dist.rank == 0 and dist.world == 1 and not args.no_cpu_baseline
    per = {}
    sharded = dist.world > 1 or args.sharded
    if sharded:
        head = bench_pr_sharded(torch, gdx, dist, args, pk)
        for a in algos:
            if a in ("tc", "bc", "sssp26"):
                per["sssp_c5" if a == "sssp26" else a] = bench_sharded_other(torch, gdx, dist,
                                                                             args, pk, a)
        algos = []  # C1 SSSP is a single-GPU config
    else:
        head = bench_pr(torch, gdx, dist, args, pk, cpu)
    for a in algos:
        if a == "sssp":
            per["sssp"] = bench_sssp(torch, gdx, dist, args, pk, 18, cpu)
        elif a == "sssp26":
            per["sssp_c5"] = bench_sssp(torch, gdx, dist, args, pk, 26, cpu and not args.no_c5_cpu)
        elif a == "tc":
            per["tc"] = bench_tc(torch, gdx, dist, args, pk, cpu)
        elif a == "bc":
            per["bc"] = bench_bc(torch, gdx, dist, args, pk, cpu)
    per["pr"] = {k: head[k] for k in ("workload", "gteps", "ms_per_step", "rounds", "roofline",
                                      "cpu_baseline", "parity", "renumbering") if k in head}
    parity = {k: v["parity"]["ok"] for k, v in per.items() if "parity" in v}
    for k, v in per.items():
        if "certificate_ok" in v:
            parity[k + "_certificate"] = v["certificate_ok"]
    line = {
        "metric": METRIC, "value": round(head["gteps"], 3), "unit": "GTEPS",
        "n_gpus": dist.world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(head["ms_per_step"], 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: counter-based RMAT generator (a,b,c,d=.57,.19,.19,.05), seed 1, built on GPU",
        "config": {"workload": head["workload"], "graph": "rmat-24", "n": head["n"], "m": head["m"],
                   "pr_rounds": head["rounds"], "damping": 0.85, "threshold": 1e-6, "max_iter": 100,
                   "parallelism": (f"vertex-range shards x{dist.world} (exchange: "
                                   f"{head.get('exchange', {}).get('kind', 'nccl')})")
                   if sharded else "single",
                   "l2": "flushed (512 MB write) before every timed step"},
        "roofline": head["roofline"], "e2e": head["e2e"], "clocks": head["clocks"],
        "gpu_launches": head["gpu_launches"], "kernels": head["kernels"],
        "parity": {"all_ok": all(parity.values()) if parity else None, **parity},
        "per_algorithm": per,
    }
    if "cpu_baseline" in head:
        line["cpu_baseline"] = head["cpu_baseline"]
    if "renumbering" in head:
        line["renumbering"] = head["renumbering"]
    if dist.rank == 0:
        print(json.dumps(line), flush=True)
    dist.close()


# ------------------------------------------------------------------ reference arm

def run_reference(args) -> None:
    """The reference's own CPU path on the headline config: interp::run(ComputePR)
    in ExecMode::Parallel on all host cores (oracle/_ref = the reference's sources
    compiled unchanged), over the same C2 graph our arm runs -- the counter-based
    RMAT-24 twin (2^28 draws, directed), its edges generated on the host by the
    oracle port (tested array-for-array against the device generator) and built
    into a CsrGraph by the reference's own buildFromEdges.  One step = one
    fixedPoint round (maxIter = 0 runs exactly one round, pr.sp:25), so the GTEPS
    (m * rounds / t) is per round like ours.  Rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import Port, Ref, ref_available
    if not ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
        return
    ref, port = Ref(), Port()
    scale = args.ref_scale
    t0 = time.perf_counter()
    u, v = port.gen_rmat_ctr(1 << scale, 16 << scale, 1, threads=CORES)
    g = ref.build(1 << scale, u, v, None, True)
    del u, v
    build_s = time.perf_counter() - t0
    times = []
    for i in range(args.warmup + args.steps):
        t1 = time.perf_counter()
        _, it = g.interp_pr(0.85, 1e-6, 0, parallel=True, threads=CORES)
        dt = time.perf_counter() - t1
        assert it == 1, it
        if i >= args.warmup:
            times.append(dt)
        print(f"reference step {i}: {dt:.2f} s", file=sys.stderr, flush=True)
    total = sum(times)
    value = g.m * len(times) / total / 1e9
    cfg = "C2" if scale == 24 else f"sample RMAT-{scale}"
    sample = (f"interp::run(ComputePR, d=0.85 tol=1e-6, maxIter=0 -> 1 fixedPoint round per "
              f"step) ExecMode::Parallel on {CORES} threads; {cfg} graph: counter-based RMAT-"
              f"{scale} twin, 2^{scale + 4} draws, directed, m={g.m}, built by the reference's "
              f"CsrGraph::buildFromEdges in {build_s:.0f}s (not timed)")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GTEPS",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": total * 1e3 / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: counter-based RMAT generator (a,b,c,d=.57,.19,.19,.05), seed 1",
        "config": {"workload": "C2 PageRank pull RMAT-24 (2^28 draws, directed) d=0.85 "
                               "tol=1e-6 (one fixedPoint round per step)" if scale == 24 else cfg,
                   "graph": f"rmat-{scale}", "m": g.m, "same_config": scale == 24,
                   "parallelism": f"{CORES} host threads"},
        "cpu_baseline": {"value": value, "unit": "GTEPS", "cores": CORES, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": value, "unit": "GTEPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def spawn_ranks(args) -> int:
    """`--gpus N` without torchrun: launch N ranks (one per GPU) through
    torch.distributed.run, or fail loudly if fewer than N GPUs are visible."""
    import socket

    import torch
    have = torch.cuda.device_count()
    if have < args.gpus:
        print(f"bench.py --gpus {args.gpus}: only {have} CUDA device(s) visible", file=sys.stderr)
        return 2
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")  # ranks / NVLS / P2P transport in the log
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def main() -> None:
    # NCCL's log (banner, INFO lines when NCCL_DEBUG is set) goes to a file, not
    # to stdout: rank 0's stdout carries exactly the one JSON line
    os.environ.setdefault("NCCL_DEBUG_FILE", os.path.join(tempfile.gettempdir(),
                                                          "gdx_nccl.%h.%p.log"))
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--algos", default="sssp,tc,bc,sssp26")
    ap.add_argument("--bc-sources", type=int, default=64)
    ap.add_argument("--ref-scale", type=int, default=24,
                    help="reference arm graph scale (24 = C2 itself)")
    ap.add_argument("--cpu-budget", type=float, default=10.0,
                    help="seconds of repeated whole CPU runs per baseline")
    ap.add_argument("--no-cpu-baseline", action="store_true",
                    help="skip the oracle parity checks and CPU baselines")
    ap.add_argument("--no-c5-cpu", action="store_true",
                    help="skip the C5 Dijkstra comparison (the device certificate still runs)")
    ap.add_argument("--sharded", action="store_true",
                    help="use the multi-GPU sharded path even at N=1 (torchrun, NCCL)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
        return
    world = os.environ.get("WORLD_SIZE")
    if world is None and args.gpus > 1:
        sys.exit(spawn_ranks(args))
    if world is not None and int(world) != args.gpus:
        sys.exit(f"bench.py --gpus {args.gpus} launched with WORLD_SIZE={world}")
    run_ours(args)


if __name__ == "__main__":
    main()
