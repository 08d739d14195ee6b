#!/bin/bash
# same-box A/B of the sharded PR path
cp paper_2401_02472_b200/lib/libgdx.so /tmp/libgdx_head.so
for v in old new old new; do
  cp variants/libgdx_$v.so paper_2401_02472_b200/lib/libgdx.so
  timeout 300 python bench.py --sharded --algos "" --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['ms_per_step'], {k:v['ms'] for k,v in d['kernels'].items()})"
done
cp /tmp/libgdx_head.so paper_2401_02472_b200/lib/libgdx.so
