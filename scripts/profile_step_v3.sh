#!/bin/bash
# ncu evidence for the bench step (run under gpurun on ONE GPU).
#  1. plain run of the exact command (must exit 0 before ncu)
#  2. launch list with per-launch device time (cold-cache, serialised) of one
#     step; M=4 microbatches so ncu finishes (same per-microbatch kernels as M=16)
#  3. --set full captures: tcgen05 GEMMs and the HBM-bound elementwise kernels
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --microbatches 4 --no-e2e --no-cpu"
$CMD > gpurun_out/plain.log 2>&1 || { echo "plain run failed"; tail -20 gpurun_out/plain.log; exit 1; }
N=$(python - <<'PY'
import json
l=[json.loads(x) for x in open("gpurun_out/plain.log") if x.startswith("{")][-1]
print(l["gpu_launches"])
PY
)
echo "launches per step: $N"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s $((3*N)) -c $N --csv \
    --log-file gpurun_out/launches_v3.csv $CMD > gpurun_out/ncu_launches.log 2>&1 || echo "launch list failed"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm2 -s 40 -c 4 \
    -o gpurun_out/prof_gemm_v3 $CMD > gpurun_out/ncu_full_gemm.log 2>&1 || echo "gemm capture failed"
# HBM-bound kernels at C2 LLM shapes, one launch each (scripts/prof_elementwise.py)
python scripts/prof_elementwise.py --json gpurun_out/elementwise_v3.jsonl > gpurun_out/prof_ew_plain.log 2>&1 || echo "elementwise plain run failed"
timeout 900 ncu --set full --clock-control none -k "regex:rmsnorm|swiglu|ce_row|sum_scale|gelu|embed" \
    -o gpurun_out/prof_ew_v3 python scripts/prof_elementwise.py --iters 1 --warm 0 > gpurun_out/ncu_full_ew.log 2>&1 || echo "elementwise capture failed"
ls -la gpurun_out | tail -8
