# the paper's head-to-head on one executor (f1) at the C4 scale: N = 4 (P = 4), M = 32, three strategies
export CUDA_DEVICE_MAX_CONNECTIONS=32
for st in bigmac memory_efficient compute_efficient; do
  echo "$st $(timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29750 \
    bench.py --gpus 4 --config C4 --microbatches 32 --steps 3 --warmup 2 --no-extra --sweep '' --no-cpu --no-e2e --strategy $st 2>&1 | grep '^{')" >> gpurun_out/strategies_c4_n4.log
done
