# the paper's head-to-head on one executor (f1) at the C4 scale: N = 4 (P = 4), M = 32, three strategies
export CUDA_DEVICE_MAX_CONNECTIONS=32
for st in bigmac memory_efficient compute_efficient; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29750 \
    bench.py --gpus 4 --config C4 --microbatches 32 --steps 2 --warmup 3 --no-extra --sweep '' --no-cpu --no-e2e --strategy $st > gpurun_out/strat_c4_$st.log 2>&1
  echo "$st $(grep '^{' gpurun_out/strat_c4_$st.log)" >> gpurun_out/strategies_c4_n4.log
done
