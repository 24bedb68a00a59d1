# A/B at N = 4 (P = 4, M = 64, C2): 1F1B vs ZB-H1, alternating, one box
export CUDA_DEVICE_MAX_CONNECTIONS=32
run() { timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 \
  --master-port $1 bench.py --gpus 4 --steps 6 --warmup 3 --no-extra --sweep '' --no-cpu --no-e2e $2 2>&1 | grep '^{' ; }
for i in 1 2; do
  echo "1f1b $(run 29610 '')" >> gpurun_out/ab_zb_n4.log
  echo "zb_h1 $(run 29620 '--llm-sched zb_h1')" >> gpurun_out/ab_zb_n4.log
done
