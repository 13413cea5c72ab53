#!/bin/bash
# step A/B of the fused kernel's L2 prefetch knobs (each argument: space-separated VAR=value list, "base" = none)
for kv in "$@"; do
  if [ "$kv" = base ]; then envs=(); else read -ra envs <<< "$kv"; fi
  for rep in 1 2; do
    env "${envs[@]}" timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-align --no-stream --no-json \
      --no-blame --no-general 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$kv', 'step', round(d['ms_per_step'], 3), 'k_fused', d['kernels']['k_fused']['ms_per_step'])"
  done
done
