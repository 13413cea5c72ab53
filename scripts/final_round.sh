#!/bin/bash
# round-closing evidence on a 4-GPU box: GPU suite + smoke + the 1-GPU profile set on GPU 0, then the
# 2- and 4-GPU bench lines and the torchrun parity cases
mkdir -p gpurun_out
CUDA_VISIBLE_DEVICES=0 timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/x_gpu_suite.txt 2>&1
echo rc=$? >> gpurun_out/x_gpu_suite.txt
CUDA_VISIBLE_DEVICES=0 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/x_smoke.txt 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 1000 bash scripts/profile_round.sh r2x > gpurun_out/x_prof.log 2>&1
echo rc=$? >> gpurun_out/x_prof.log
for N in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29531 \
    bench.py --gpus $N > gpurun_out/x_b${N}.json 2> gpurun_out/x_b${N}.err
  echo "N=$N rc=$?" >> gpurun_out/x_prof.log
done
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -p no:cacheprovider > gpurun_out/x_multi_tests.txt 2>&1
