# N = 4 default config: encoder ops on their own stream (BM_ENC_STREAM=1) vs on the compute stream
export CUDA_DEVICE_MAX_CONNECTIONS=32
run() { timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 \
  --master-port $1 bench.py --gpus 4 --steps 6 --warmup 3 --no-extra --sweep '' --no-cpu --no-e2e 2>&1 | grep '^{' ; }
for i in 1 2; do
  echo "compute $(BM_ENC_STREAM=0 run 29610)" >> gpurun_out/ab_encstream.log
  echo "encstream $(BM_ENC_STREAM=1 run 29620)" >> gpurun_out/ab_encstream.log
done
