# C3 (interleaved, V = 2) at N = 4: generator / encoder on the lightest rank vs everywhere
export CUDA_DEVICE_MAX_CONNECTIONS=32
run() { timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 \
  --master-port $1 bench.py --gpus 4 --config C3 --steps 4 --warmup 3 --no-extra --sweep '' --no-cpu --no-e2e $2 2>&1 | grep '^{' ; }
for i in 1 2; do
  echo "light $(run 29610 '')" >> gpurun_out/ab_c3.log
  echo "all $(run 29620 '--gen-exclude none --enc-exclude none')" >> gpurun_out/ab_c3.log
done
