# half-layer partition: multi-GPU parity (NCCL, one GPU per rank), then A/B at N = 4 (C2, P = 4, M = 64)
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29502 tests/mp_step.py C1:2:4:1:f32:dp_shard+halves3-5:1 C1:2:4:1:bf16:dp_shard+halves5-3:1 C1M:2:4:1:bf16:dp_shard+halves3-5:1:gm2 C1:2:4:1:f32:dp_shard+halves3-5+zb:1 C1:2:8:2:f32:dp_shard+halves1-3-2-2:1 > gpurun_out/halves_mr2.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29504 tests/mp_step.py C1:4:8:1:f32:dp_shard+halves3-2-2-1:1 C1:4:8:1:bf16:dp_shard+halves1-1-1-5+zb+edge:1 C1:2:4:1:f32:dp_shard+halves3-5:2 > gpurun_out/halves_mr4.log 2>&1
grep -h "CASE" gpurun_out/halves_mr*.log
run() { timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 \
  --master-port $1 bench.py --gpus 4 --steps 6 --warmup 3 --no-extra --sweep '' --no-cpu --no-e2e $2 2>&1 | grep '^{' ; }
for i in 1 2; do
  echo "layers $(run 29610 '')" >> gpurun_out/ab_halves_n4.log
  echo "halves $(run 29620 '--partition halves')" >> gpurun_out/ab_halves_n4.log
  echo "halves_zb $(run 29630 '--partition halves --llm-sched zb_h1')" >> gpurun_out/ab_halves_n4.log
done
