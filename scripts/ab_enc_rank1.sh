# N = 4: encoder on rank 1 (own stream) vs on rank 3 (default); generator on rank 3
export CUDA_DEVICE_MAX_CONNECTIONS=32
run() { timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 \
  --master-port $1 bench.py --gpus 4 --steps 6 --warmup 3 --no-extra --sweep '' --no-cpu --no-e2e $2 2>&1 | grep '^{' ; }
for i in 1 2; do
  echo "enc3 $(run 29610 '')" >> gpurun_out/ab_enc_rank1.log
  echo "enc1 $(run 29620 '--enc-exclude 0,2,3')" >> gpurun_out/ab_enc_rank1.log
done
