#!/bin/bash
# Timing / traffic experiment on the GPU box: DRAM bytes and time of k_fused_t with the shipped library,
# then with the library rebuilt in the box's scratch copy under -DMS_EXP_SKIP=<bits> for each argument
# (results of those builds are invalid by construction; never run this in a tree you ship from).
set -u
m="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_write.sum"
run() {
  /usr/local/cuda/bin/ncu --metrics $m --clock-control none -k regex:k_fused_t -c 1 --csv python bench.py --steps 1 --warmup 1 \
    --no-cpu --no-e2e --no-align --no-stream --no-json --no-blame --no-general 2>/dev/null | grep '"k_fused_t\|k_fused_t<' | \
    awk -F'","' -v t="$1" '{print t, $(NF-2), $NF}'
}
run base
for bits in "$@"; do
  MS_NVCC_EXTRA="-DMS_EXP_SKIP=$bits" python -c "import paper_2507_19845_b200._build as b; b.build(force=True)" > /dev/null 2>&1
  run "skip$bits"
done
