#!/bin/bash
# L2 fetch-granularity experiment: k_fused_t / k_cross_reduce DRAM bytes and time for each MS_L2_FETCH value
m="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
for v in "$@"; do
  MS_L2_FETCH=$v /usr/local/cuda/bin/ncu --metrics $m --clock-control none -k regex:"k_fused_t|k_cross_reduce" -c 2 --csv python bench.py \
    --steps 1 --warmup 1 --no-cpu --no-e2e --no-align --no-stream --no-json --no-blame --no-general 2>/dev/null | python scripts/ncu_metrics.py fetch$v
done
