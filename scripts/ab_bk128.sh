# 128-deep K blocks: parity tests, GEMM A/B, C2 step A/B
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "bk128" > gpurun_out/bk128_tests.log 2>&1
tail -3 gpurun_out/bk128_tests.log
if grep -q " passed" gpurun_out/bk128_tests.log && ! grep -q "failed\|error" gpurun_out/bk128_tests.log; then
  timeout 900 python scripts/gemm_ab_knob.py 3 bk128 > gpurun_out/bk128_knob.log 2>&1
  for v in 0 1 0 1; do
    echo "BK128=$v $(BM_GEMM_BK128=$v timeout 300 python bench.py --steps 6 --warmup 3 --no-extra --sweep '' --no-cpu --no-e2e 2>&1 | grep '^{')" >> gpurun_out/bk128_step.log
  done
fi
