mkdir -p gpurun_out
CUDA_VISIBLE_DEVICES=0 bash scripts/exp_env.sh base MS_FT_PF_OWN=0 MS_FT_PF=148 MS_FT_PF=74 MS_TILE_ORDER=0 MS_FT_PF_P2P=0 > gpurun_out/env.log 2>&1
for N in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29521 \
    bench.py --gpus $N > gpurun_out/mg2_b${N}.json 2> gpurun_out/mg2_b${N}.err
  echo "N=$N rc=$?"
done
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -p no:cacheprovider > gpurun_out/mg2_tests.txt 2>&1
echo "tests rc=$?"
