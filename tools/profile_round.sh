#!/bin/bash
# One GPU call that produces this round's evidence under gpurun_out/:
# the bench line, the ncu launch list of the headline bench command, and one
# `ncu --set full` capture per hot kernel (tools/kernel_driver.py drives the
# BASELINE configs).  Summarise with tools/make_profiles.py afterwards.
set -u
O=gpurun_out
mkdir -p $O
timeout 900 python bench.py > $O/bench_round.json 2> $O/bench_round.err
echo "bench rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $O/launches_pr.csv python bench.py --algos "" --steps 2 --warmup 3 \
    --no-cpu-baseline > $O/launches_bench.log 2>&1
echo "launch list rc=$?"
cap() {  # name algo kernel-regex skip   (kernels inside a CUDA graph with conditional
         # nodes cannot be profiled one by one: SSSP captures use the host-driven loop,
         # GDX_SSSP_MODE=scan, which runs the same kernels)
    GDX_SSSP_MODE=scan timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$3" -s "$4" -c 1 \
        -o $O/ncu_$1 -f python tools/kernel_driver.py --algo "$2" --reps 2 > $O/ncu_$1.log 2>&1
    echo "ncu $1 rc=$?"
}
cap pr_edges pr k_pr_edges 2
cap pr_vertices pr k_pr_vertices 2
cap tc tc k_tc_oriented 0
cap sssp_c1_relax sssp k_sssp_scan_relax 3
cap sssp_c5_relax sssp26 k_sssp_scan_relax 3
cap bc bc k_bc_cta 0
