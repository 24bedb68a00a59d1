# N = 4, C2, halves, 1F1B: encoder on every stage vs on the lightest stage only (generator on the lightest)
export CUDA_DEVICE_MAX_CONNECTIONS=32
run() { timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 \
  --master-port $1 bench.py --gpus 4 --steps 6 --warmup 3 --no-extra --sweep '' --no-cpu --no-e2e $2 2>&1 | grep '^{' ; }
for i in 1 2; do
  echo "enc_all $(run 29610 '--enc-exclude none')" >> gpurun_out/ab_enc_n4.log
  echo "enc_light $(run 29620 '--enc-exclude 0,1,2')" >> gpurun_out/ab_enc_n4.log
done
