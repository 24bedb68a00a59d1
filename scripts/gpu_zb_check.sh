set -x
export CUDA_DEVICE_MAX_CONNECTIONS=32
python -m pytest tests/test_gpu_step.py -q -x -k "zb_h1" 2>&1 | tail -5 > gpurun_out/zb_single.log
export BM_TEST_ONE_GPU=1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29502 tests/mp_step.py C1:2:4:1:f32:dp_shard+zb:1 C1:2:4:1:bf16:dp_shard+zb:1 C1M:2:4:1:bf16:dp_shard+zb:1:gm2 C1:2:4:1:f32:entry_stage+last_stage+zb:1 > gpurun_out/zb_mr2.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29504 tests/mp_step.py C1:4:8:1:f32:dp_shard+zb:1 C1:4:16:1:bf16:dp_shard+zb:1 C1:4:8:1:f32:last_stage+zb+edge:1 C1M:4:8:1:bf16:dp_shard+zb+fsdp:1:gm2 C1:2:4:1:f32:dp_shard+zb:2 > gpurun_out/zb_mr4.log 2>&1
unset BM_TEST_ONE_GPU
timeout 300 python bench.py --steps 5 --warmup 3 --no-extra --sweep '' --no-cpu --llm-sched zb_h1 > gpurun_out/zb_bench_n1.log 2>&1
timeout 300 python bench.py --steps 5 --warmup 3 --no-extra --sweep '' --no-cpu > gpurun_out/base_bench_n1.log 2>&1
grep -h "CASE\|passed\|failed" gpurun_out/zb_*.log
