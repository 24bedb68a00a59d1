#!/bin/bash
# ncu evidence for the bench step, round 2 (ONE GPU, under gpurun):
#  1. plain run of the exact command (must exit 0 before ncu)
#  2. launch list with per-launch device time of one C2 step (M = 16, the bench's
#     workload; cold-cache, serialised: shares, not absolutes)
#  3. --set full of CTA-pair GEMM launches of the step (traffic for bench.py)
#  4. --set full of the HBM-bound elementwise kernels at C2 shapes
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-extra"
$CMD > gpurun_out/plain.log 2>&1 || { echo "plain run failed"; tail -20 gpurun_out/plain.log; exit 1; }
N=$(python -c 'import json;l=[json.loads(x) for x in open("gpurun_out/plain.log") if x.startswith("{")][-1];print(l["gpu_launches"])')
echo "launches per step: $N"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -s $((3*N)) -c $N --csv \
    --log-file gpurun_out/launches_r02.csv $CMD > gpurun_out/ncu_launches.log 2>&1 || echo "launch list failed"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm2 -s 100 -c 6 \
    -o gpurun_out/prof_gemm_r02 $CMD > gpurun_out/ncu_full_gemm.log 2>&1 || echo "gemm capture failed"
python scripts/prof_elementwise.py --json gpurun_out/elementwise_r02.jsonl > gpurun_out/prof_ew_timed.log 2>&1 || echo "elementwise timed run failed"
python scripts/prof_elementwise.py --iters 1 --warm 0 > gpurun_out/prof_ew_plain.log 2>&1 &&
timeout 900 ncu --set full --clock-control none -k "regex:rmsnorm|swiglu|ce_row|gelu|embed" \
    -o gpurun_out/prof_ew_r02 python scripts/prof_elementwise.py --iters 1 --warm 0 > gpurun_out/ncu_full_ew.log 2>&1 || echo "elementwise capture failed"
ls -la gpurun_out | tail -8
