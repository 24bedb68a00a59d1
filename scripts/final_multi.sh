# end-of-round multi-GPU check on 4 GPUs: every multi-rank parity case over NCCL (one GPU per rank),
# then the default bench lines at N = 4 and N = 2 and C3 at N = 4
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 2400 python -m pytest tests/test_gpu_step.py -q -k "multirank or timeout" > gpurun_out/pytest_multirank_4gpu_final.log 2>&1
tail -2 gpurun_out/pytest_multirank_4gpu_final.log
for N in 4 2; do
  timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 \
    --master-port $((29700 + N)) bench.py --gpus $N > gpurun_out/bench_n${N}_final.log 2>&1
done
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 \
  --master-port 29720 bench.py --gpus 4 --config C3 --no-extra --sweep '' > gpurun_out/bench_c3_n4_final.log 2>&1
