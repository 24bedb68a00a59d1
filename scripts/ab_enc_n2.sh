# N = 2: encoder on both ranks (default) vs on rank 1 with its own stream
export CUDA_DEVICE_MAX_CONNECTIONS=32
run() { timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 \
  --master-port $1 bench.py --gpus 2 --steps 6 --warmup 3 --no-extra --sweep '' --no-cpu --no-e2e $2 2>&1 | grep '^{' ; }
for i in 1 2; do
  echo "both $(run 29610 '')" >> gpurun_out/ab_enc_n2.log
  echo "rank1_stream $(run 29620 '--enc-exclude 0')" >> gpurun_out/ab_enc_n2.log
done
