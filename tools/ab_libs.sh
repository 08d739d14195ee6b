#!/bin/bash
# Same-box A/B of library variants (variants/libgdx_<name>.so): each
# variant in turn replaces lib/libgdx.so in this (scratch) copy of the repo and
# runs `bench.py --algos <algos>`; prints the per-algorithm kernel time.
# A variant may carry environment settings: <name>[:VAR=value[,VAR=value]].
#   tools/ab_libs.sh "bc" head xf head xf
#   tools/ab_libs.sh "sssp26" head head:GDX_SSSP_NARROW=0
set -u
algos=$1; shift
cp paper_2401_02472_b200/lib/libgdx.so /tmp/libgdx_head.so
for spec in "$@"; do
    v=${spec%%:*}
    envs=""
    [ "$spec" != "$v" ] && envs=$(echo "${spec#*:}" | tr ',' ' ')
    if [ "$v" = head ]; then cp /tmp/libgdx_head.so paper_2401_02472_b200/lib/libgdx.so
    else cp variants/libgdx_$v.so paper_2401_02472_b200/lib/libgdx.so; fi
    env $envs timeout 600 python bench.py --algos "$algos" --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json, sys
d = json.loads(sys.stdin.read())
for k, x in d['per_algorithm'].items():
    if k != 'pr' or '$algos' == '':
        r = x.get('roofline', {})
        print('$spec', k, round(x['ms_per_step'], 3), 'kernel_ms', r.get('kernel_ms_per_unit'), 'frac', r.get('frac'))
"
done
cp /tmp/libgdx_head.so paper_2401_02472_b200/lib/libgdx.so
