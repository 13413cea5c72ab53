#!/bin/bash
# environment-variable experiment: k_fused_t (and k_cross_reduce) time / DRAM bytes under ncu, then the
# bench step time, for each "VAR=value" argument (one at a time; "base" = none)
m="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
for kv in "$@"; do
  if [ "$kv" = base ]; then envs=(); else envs=("$kv"); fi
  env "${envs[@]}" /usr/local/cuda/bin/ncu --metrics $m --clock-control none -k regex:"k_fused_t" -c 1 --csv python bench.py \
    --steps 1 --warmup 1 --no-cpu --no-e2e --no-align --no-stream --no-json --no-blame --no-general 2>/dev/null | python scripts/ncu_metrics.py "$kv"
  env "${envs[@]}" timeout -s KILL 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-align --no-stream --no-json \
    --no-blame --no-general 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$kv', 'step', round(d['ms_per_step'], 3), {k: v['ms_per_step'] for k, v in d['kernels'].items() if v['ms_per_step'] > 0.05})"
done
