set -x
mkdir -p gpurun_out
for N in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 \
    bench.py --gpus $N > gpurun_out/mg_b${N}.json 2> gpurun_out/mg_b${N}.err
  echo "N=$N rc=$?"
done
MS_SHARD_PROFILE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 \
  bench.py --gpus 4 --steps 5 --warmup 3 > gpurun_out/mg_b4_prof.json 2> gpurun_out/mg_b4_prof.err
echo "prof rc=$?"
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -p no:cacheprovider > gpurun_out/mg_tests.txt 2>&1
echo "tests rc=$?"
