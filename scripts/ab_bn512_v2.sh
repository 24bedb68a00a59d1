# 256x512 vs 256x256 with 128-deep K blocks (the new default for 256-wide tiles)
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 900 python scripts/gemm_ab_knob.py 3 bn512 > gpurun_out/bn512_v2_knob.log 2>&1
