#!/bin/bash
# A/B timing of two in-tree builds (libmegascan.so vs $1, e.g. paper_2507_19845_b200/libmegascan_ab.so), alternating,
# bench step and kernel breakdown (no ncu)
for rep in 1 2; do
  for lib in "" "$1"; do
    MEGASCAN_LIB=$lib timeout -s KILL 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-align --no-stream --no-json \
      --no-blame --no-general 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('${lib:-current}', 'step', round(d['ms_per_step'], 3), {k: v['ms_per_step'] for k, v in d['kernels'].items() if v['ms_per_step'] > 0.05})"
  done
done
