export CUDA_DEVICE_MAX_CONNECTIONS=32
for sch in auto zb_h1; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29660 \
  scripts/trace_step.py --M 64 --stage-layers 9,9,9,5 --halves --gen-exclude 7 --enc-exclude 7 --llm-sched $sch \
  --out gpurun_out/trace_n4_final_$sch.json > gpurun_out/trace_n4_final_$sch.txt 2>&1
done
