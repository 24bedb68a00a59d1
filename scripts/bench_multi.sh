# default bench lines at N = 4 and N = 2 (and N = 1) on one box, as the driver launches them
export CUDA_DEVICE_MAX_CONNECTIONS=32
for N in 4 2; do
  start=$(date +%s)
  timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 \
    --master-port $((29700 + N)) bench.py --gpus $N > gpurun_out/bench_n${N}_default.log 2>&1
  echo "N=$N wall $(( $(date +%s) - start )) s" >> gpurun_out/bench_multi_wall.log
done
