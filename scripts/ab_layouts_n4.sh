# N = 4 C2: pipeline layouts P = 4, P = 2 x D = 2, P = 1 x D = 4 (default bench otherwise)
export CUDA_DEVICE_MAX_CONNECTIONS=32
run() { timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 \
  --master-port $1 bench.py --gpus 4 --steps 6 --warmup 3 --no-extra --sweep '' --no-cpu --no-e2e $2 2>&1 | grep '^{' ; }
echo "P4 $(run 29610 '')" >> gpurun_out/ab_layouts_n4.log
echo "P2D2 $(run 29620 '--stages 2')" >> gpurun_out/ab_layouts_n4.log
echo "P1D4 $(run 29630 '--stages 1')" >> gpurun_out/ab_layouts_n4.log
echo "P4zb $(run 29640 '--llm-sched zb_h1')" >> gpurun_out/ab_layouts_n4.log
