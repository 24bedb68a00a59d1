# N = 2 (C2, P = 2, M = 32): where the encoder / generator run, 1F1B; plus a per-op trace of the default
export CUDA_DEVICE_MAX_CONNECTIONS=32
run() { timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 \
  --master-port $1 bench.py --gpus 2 --steps 6 --warmup 3 --no-extra --sweep '' --no-cpu --no-e2e $2 2>&1 | grep '^{' ; }
echo "default $(run 29610 '')" >> gpurun_out/ab_n2.log
echo "noexcl $(run 29620 '--gen-exclude none --enc-exclude none')" >> gpurun_out/ab_n2.log
echo "genx0 $(run 29630 '--enc-exclude none')" >> gpurun_out/ab_n2.log
echo "encx0 $(run 29640 '--gen-exclude none')" >> gpurun_out/ab_n2.log
echo "layers $(run 29650 '--partition layers')" >> gpurun_out/ab_n2.log
for sch in auto zb_h1; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29660 \
  scripts/trace_step.py --M 32 --stage-layers 18,14 --halves --gen-exclude 1 --enc-exclude 1 --llm-sched $sch \
  --out gpurun_out/trace_n2_$sch.json > gpurun_out/trace_n2_$sch.txt 2>&1
done
