#!/bin/bash
# A/B of the tile order of the general path and blame kernels (MS_TILE_ORDER=0: rank-major index
# order, 1: interleaved across ranks)
for v in 0 1; do
  MS_TILE_ORDER=$v python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --no-stream --no-json --no-align 2>/dev/null | tail -1 > gpurun_out/to_$v.json
  python -c "
import json; d=json.load(open('gpurun_out/to_$v.json')); g=d['general_path']; b=d['blame']
print('order=$v', d['ms_per_step'], g['forced']['ms_per_step'], g['one_violation']['ms_per_step'], 'blame', b['ms_per_call'], {k: v['ms_per_call'] for k, v in b['kernels'].items()})"
done
