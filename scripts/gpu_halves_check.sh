export CUDA_DEVICE_MAX_CONNECTIONS=32
export BM_TEST_ONE_GPU=1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29502 tests/mp_step.py C1:2:4:1:f32:dp_shard+halves3-5:1 C1:2:4:1:bf16:dp_shard+halves5-3:1 C1M:2:4:1:bf16:dp_shard+halves3-5:1:gm2 C1:2:4:1:f32:dp_shard+halves3-5+zb:1 C1:2:8:2:f32:dp_shard+halves1-3-2-2:1 > gpurun_out/halves_mr2.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29504 tests/mp_step.py C1:4:8:1:f32:dp_shard+halves3-2-2-1:1 C1:4:8:1:bf16:dp_shard+halves1-1-1-5+zb+edge:1 C1:2:4:1:f32:dp_shard+halves3-5:2 > gpurun_out/halves_mr4.log 2>&1
grep -h "CASE" gpurun_out/halves_mr*.log
