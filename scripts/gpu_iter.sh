#!/bin/bash
# one development iteration on the GPU box: parity check, C3-100 kernel times, full-C3 bench, ncu of k_stage
tag=${1:-x}
timeout -s KILL 400 python scripts/dev_check.py > gpurun_out/dev_$tag.txt 2>&1; echo "dev rc=$?"; cat gpurun_out/dev_$tag.txt
python scripts/prof_case.py 100 > gpurun_out/p_$tag.txt 2>&1; cat gpurun_out/p_$tag.txt
timeout -s KILL 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-align --no-stream --no-json --no-blame > gpurun_out/b_$tag.json 2> gpurun_out/b_$tag.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/b_$tag.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['roofline']['frac'], d['roofline']['dominant_kernel']); print({k: v['ms_per_step'] for k, v in d['kernels'].items()})"
if [ "$2" != "noprof" ]; then
timeout -s KILL 600 /usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:k_stage -s 1 -c 1 -o gpurun_out/k_stage_$tag python scripts/prof_case.py 100 > gpurun_out/ncu_$tag.log 2>&1; tail -1 gpurun_out/ncu_$tag.log
fi
