# exercise the C5 sweep code path at P = 4 (the driver runs it at N = 8 with P = 8)
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29740 \
  bench.py --gpus 4 --steps 3 --warmup 3 --no-cpu --no-e2e --sweep '' --no-c4-strong --c5 --c5-stages 4 --c5-sweep 8,16,32,64 \
  > gpurun_out/bench_c5_p4.log 2>&1
tail -c 2500 gpurun_out/bench_c5_p4.log
