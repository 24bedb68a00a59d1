#!/bin/bash
# ncu evidence for the bench step (run under gpurun on ONE GPU).
#  1. plain run of the exact command (must exit 0 before ncu)
#  2. launch list with per-launch device time (cold-cache, serialised) of one
#     step; M=4 microbatches so ncu finishes (same per-microbatch kernels as M=16)
#  3. --set full capture of a few tcgen05 GEMM launches
set -e
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --microbatches 4 --no-e2e --no-cpu"
$CMD > gpurun_out/plain.log 2>&1
N=$(python - <<'PY'
import json
l=[json.loads(x) for x in open("gpurun_out/plain.log") if x.startswith("{")][-1]
print(l["gpu_launches"])
PY
)
echo "launches per step: $N"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s $((3*N)) -c $N --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1 || true
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm -s 40 -c 4 \
    -o gpurun_out/prof_gemm $CMD > gpurun_out/ncu_full.log 2>&1 || true
ls -la gpurun_out
