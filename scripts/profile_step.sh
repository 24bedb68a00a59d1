#!/bin/bash
# ncu evidence for the bench step (run under gpurun on ONE GPU).
#  1. plain run of the exact command (must exit 0 before ncu)
#  2. launch list with per-launch device time (cold-cache, serialised)
#  3. --set full capture of a few tcgen05 GEMM launches
set -e
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu"
$CMD > gpurun_out/plain.log 2>&1
# skip the 3 warm-up steps (~6600 launches each), list one full step
ncu --metrics gpu__time_duration.sum --clock-control none -s 19800 -c 6700 --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1 || true
ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 40 -c 6 \
    -o gpurun_out/prof_gemm $CMD > gpurun_out/ncu_full.log 2>&1 || true
ls -la gpurun_out
