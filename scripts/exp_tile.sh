#!/bin/bash
# A/B of the transposed fused kernel's CTA size (compile-time MS_FT_NT) and tile positions (MS_FT_T):
# each argument "NT:T" rebuilds the library in the box's scratch copy, times the step (k_fused_t and the
# step ms) and runs the bench-shape parity cases under the same setting. "NT:-" keeps the default T.
set -u
for v in "$@"; do
  nt=${v%%:*}; t=${v##*:}
  MS_NVCC_EXTRA="-DMS_FT_NT=$nt" python -c "import paper_2507_19845_b200._build as b; b.build(force=True)" > /dev/null 2>&1
  if [ "$t" = "-" ]; then unset MS_FT_T; else export MS_FT_T=$t; fi
  python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-align --no-stream --no-json --no-blame --no-general \
    2> gpurun_out/tile_${nt}_${t}.err | tail -1 > gpurun_out/tile.json
  python -c "
import json; d=json.load(open('gpurun_out/tile.json'))
print('$v', 'step', round(d['ms_per_step'], 3), {k: v['ms_per_step'] for k, v in d['kernels'].items() if v['ms_per_step'] > 0.05})"
  grep -m1 "MS_FT_T" gpurun_out/tile_${nt}_${t}.err
  timeout 600 python -m pytest tests/test_gpu_benchshape.py -x -q -p no:cacheprovider -k "c3_shape or u32" 2>&1 | tail -1
done
