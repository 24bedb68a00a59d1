export CUDA_DEVICE_MAX_CONNECTIONS=32
export BM_TEST_ONE_GPU=1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29504 tests/mp_step.py C1:4:8:1:bf16:dp_shard+halves3-2-2-1+genx7+encx7:1:es C1:4:8:1:f32:dp_shard+halves3-2-2-1+genx7+encx7+zb:1:es > gpurun_out/es_mr4.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29502 tests/mp_step.py C1:2:4:1:f32:dp_shard+encx1:1:es > gpurun_out/es_mr2.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=8 --master-addr 127.0.0.1 --master-port 29508 tests/mp_step.py C1:4:8:1:bf16:dp_shard+halves3-2-2-1+genx7+encx7:2:es > gpurun_out/es_mr8.log 2>&1
grep -h CASE gpurun_out/es_mr*.log
