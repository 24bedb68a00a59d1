export CUDA_DEVICE_MAX_CONNECTIONS=32
export BM_TEST_ONE_GPU=1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29504 tests/mp_step.py C1:4:8:1:bf16:dp_shard+halves3-2-2-1+genx7+encx7:1 C1:4:8:1:f32:dp_shard+halves3-2-2-1+genx7+encx7+zb:1 C1:2:4:1:bf16:dp_shard+halves5-3+genx1+encx1:2 > gpurun_out/defaults_mr.log 2>&1
grep -h CASE gpurun_out/defaults_mr.log
