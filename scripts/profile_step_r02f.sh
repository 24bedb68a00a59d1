#!/bin/bash
# ncu evidence of the bench step at the end of round 2 (ONE GPU, under gpurun):
#  1. plain run of the exact command (must exit 0 before ncu)
#  2. launch list with per-launch device time of one C2 step (cold-cache, serialised: shares)
#  3. --set full of the forward and backward CTA-pair GEMMs of one layer (traffic for bench.py)
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-extra --sweep ''"
eval $CMD > gpurun_out/plain_f.log 2>&1 || { echo "plain run failed"; tail -20 gpurun_out/plain_f.log; exit 1; }
N=$(python -c 'import json;l=[json.loads(x) for x in open("gpurun_out/plain_f.log") if x.startswith("{")][-1];print(l["gpu_launches"])')
echo "launches per step: $N"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -s $((3*N)) -c $N --csv \
    --log-file gpurun_out/launches_r02f.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-extra --sweep '' > gpurun_out/ncu_launches_f.log 2>&1 || echo "launch list failed"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm2 -s 100 -c 6 \
    -o gpurun_out/prof_gemm_fwd_r02f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-extra --sweep '' > gpurun_out/ncu_full_fwd_f.log 2>&1 || echo "fwd capture failed"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm2 -s 35 -c 8 \
    -o gpurun_out/prof_gemm_bwd_r02f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-extra --sweep '' > gpurun_out/ncu_full_bwd_f.log 2>&1 || echo "bwd capture failed"
ls -la gpurun_out | tail -6
