# SwiGLU forward with 128-deep K blocks: parity, standalone A/B, C2 step A/B; new bn512 model in the step
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "swiglu or bk128 or bn512" > gpurun_out/swbk_tests.log 2>&1
tail -1 gpurun_out/swbk_tests.log
if ! grep -q "failed\|error" gpurun_out/swbk_tests.log; then
  timeout 900 python scripts/gemm_ab_knob.py 3 swiglu_bk128 2>&1 | head -2 > gpurun_out/swbk_knob.log
  for v in 0 1 0 1; do
    echo "SWBK=$v $(BM_GEMM_SWIGLU_BK128=$v timeout 300 python bench.py --steps 6 --warmup 3 --no-extra --sweep '' --no-cpu --no-e2e 2>&1 | grep '^{')" >> gpurun_out/swbk_step.log
  done
fi
