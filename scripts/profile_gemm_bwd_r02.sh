#!/bin/bash
# ncu --set full of the backward CTA-pair GEMMs of the C2 step (first two layers of
# B(0): down wgrad, down dgrad + SwiGLU backward, gate_up wgrad, gate_up dgrad; the
# first 35 pair launches are F(0): 16 x (gate_up, down) + the LM head's three)
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-extra"
$CMD > gpurun_out/plain_bwd.log 2>&1 || { echo "plain run failed"; tail -20 gpurun_out/plain_bwd.log; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm2 -s 35 -c 8 \
    -o gpurun_out/prof_gemm_bwd_r02 $CMD > gpurun_out/ncu_full_gemm_bwd.log 2>&1 || echo "gemm bwd capture failed"
