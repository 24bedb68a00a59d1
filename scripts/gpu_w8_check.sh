# world-8 multi-rank parity (the N = 8 bench shape: P = 4 x D = 2) with all ranks on one GPU
export CUDA_DEVICE_MAX_CONNECTIONS=32
export BM_TEST_ONE_GPU=1
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node=8 --master-addr 127.0.0.1 --master-port 29508 \
  tests/mp_step.py C1:4:8:1:bf16:dp_shard+halves3-2-2-1+genx7+encx7:2 C1:4:8:1:f32:dp_shard+halves3-2-2-1+genx7+encx7+zb:2 \
  > gpurun_out/w8_mr.log 2>&1
grep -h CASE gpurun_out/w8_mr.log; tail -3 gpurun_out/w8_mr.log
