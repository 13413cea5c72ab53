#!/bin/bash
# round profile set (B200_PROFILING.md recipe): default bench line, the launch list of the same command
# under ncu (per-launch gpu__time_duration, cold-cache, serialised), and one --set full capture of the
# dominant kernel for its DRAM traffic and issue metrics. Each ncu pass runs after the plain command
# exited 0.
tag=${1:-r2}
set -e
python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-align --no-stream --no-json --no-blame --no-general \
  > gpurun_out/${tag}_short.json 2> gpurun_out/${tag}_short.err
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${tag}_launches_c3.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-align \
  --no-stream --no-json --no-blame --no-general > gpurun_out/${tag}_ncu_launch.log 2>&1
/usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:k_fused_t -c 1 \
  --csv --page raw --log-file gpurun_out/${tag}_k_fused_t_raw.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e \
  --no-align --no-stream --no-json --no-blame --no-general > gpurun_out/${tag}_ncu_full.log 2>&1
echo done
