#!/bin/bash
# One GPU call that produces a round's evidence under gpurun_out/: the bench
# line, the ncu launch list of the headline bench command, DRAM bytes per unit
# of work (SSSP/TC/BC call, PR round) for roofline.traffic, and one
# `ncu --set full` capture per hot kernel (tools/kernel_driver.py drives the
# BASELINE configs).  Summarise with tools/make_profiles.py /
# tools/ncu_unit_traffic.py afterwards.
set -u
O=gpurun_out
mkdir -p $O
R=${1:-r02}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $O/launches_pr_$R.csv python bench.py --algos "" --steps 2 --warmup 3 \
    --no-cpu-baseline > $O/launches_bench_$R.log 2>&1
echo "launch list rc=$?"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
# C2 / C5 run on the renumbered graph from the second call on (csrc/relabel.cu);
# GDX_RELABEL=1 makes every captured call use it (the bench's timed calls do)
traffic() {  # name algo kernel-regex [VAR=value ...]
    env GDX_SSSP_MODE=scan ${@:4} timeout 900 ncu --metrics $M --clock-control none -k "regex:$3" --csv \
        --log-file $O/traffic_$1_$R.csv python tools/kernel_driver.py --algo "$2" --reps 2 \
        > $O/traffic_$1_$R.log 2>&1
    echo "traffic $1 rc=$?"
}
traffic sssp_c1 sssp k_sssp
traffic sssp_c5 sssp26 k_sssp GDX_RELABEL=1
traffic pr pr "k_pr_(edges|cross|vertices)" GDX_RELABEL=1
traffic tc tc k_tc
traffic bc bc k_bc
cap() {  # name algo kernel-regex skip [VAR=value ...]
    env GDX_SSSP_MODE=scan ${@:5} timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$3" -s "$4" -c 1 \
        -o $O/ncu_$1_$R -f python tools/kernel_driver.py --algo "$2" --reps 2 > $O/ncu_$1_$R.log 2>&1
    echo "ncu $1 rc=$?"
}
cap pr_edges pr k_pr_edges 2 GDX_RELABEL=1
cap pr_vertices pr k_pr_vertices 2 GDX_RELABEL=1
cap tc tc k_tc_oriented 0
cap sssp_relax_c1 sssp k_sssp_scan_relax 3
# the third round's main relaxation (the largest of a C5 call; main and small-vertex
# launches alternate)
cap sssp_relax sssp26 k_sssp_scan_relax 4 GDX_RELABEL=1
cap bc_cta bc k_bc_cta 0
