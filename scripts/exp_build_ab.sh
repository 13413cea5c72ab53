#!/bin/bash
# A/B of compile-time variants on the GPU box: for each argument (extra nvcc flags, "base" = none) the
# library is rebuilt in the box's scratch copy and one bench section timed (SECTION=general | align | blame; blame also prints the step kernels).
set -u
sec=${SECTION:-general}
for fl in "$@"; do
  if [ "$fl" = base ]; then ex=""; else ex="$fl"; fi
  MS_NVCC_EXTRA="$ex" python -c "import paper_2507_19845_b200._build as b; b.build(force=True)" > /dev/null 2>&1
  if [ "$sec" = blame ]; then
    python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --no-stream --no-json --no-align --no-general 2>/dev/null | tail -1 > gpurun_out/ab.json
    python -c "
import json; d=json.load(open('gpurun_out/ab.json')); b=d['blame']
print('$fl', round(d['ms_per_step'], 3), {k: v['ms_per_step'] for k, v in d['kernels'].items() if v['ms_per_step'] > 0.05}, 'blame', round(b['ms_per_call'], 2), {k: v['ms_per_call'] for k, v in b['kernels'].items()})"
  elif [ "$sec" = align ]; then
    python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --no-stream --no-json --no-blame --no-general 2>/dev/null | tail -1 > gpurun_out/ab.json
    python -c "
import json; d=json.load(open('gpurun_out/ab.json')); a=d['alignment']
print('$fl', round(d['ms_per_step'], 3), round(a['ms_per_call'], 2), {k: v['ms_per_call'] for k, v in a['kernels'].items()})"
  else
    python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --no-stream --no-json --no-align --no-blame 2>/dev/null | tail -1 > gpurun_out/ab.json
    python -c "
import json; d=json.load(open('gpurun_out/ab.json')); g=d['general_path']
print('$fl', round(d['ms_per_step'], 3), round(g['forced']['ms_per_step'], 2), g['forced']['kernels_ms'])"
  fi
done
