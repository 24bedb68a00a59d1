# two-pair clusters with A multicast: parity tests, GEMM A/B, C2 step A/B
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "cluster4" > gpurun_out/cl4_tests.log 2>&1
tail -3 gpurun_out/cl4_tests.log
if grep -q " passed" gpurun_out/cl4_tests.log && ! grep -q "failed\|error" gpurun_out/cl4_tests.log; then
  timeout 900 python scripts/gemm_ab_knob.py 3 cl4 > gpurun_out/cl4_knob.log 2>&1
  for v in 0 1 0 1; do
    echo "CL4=$v $(BM_GEMM_CL4=$v timeout 300 python bench.py --steps 6 --warmup 3 --no-extra --sweep '' --no-cpu --no-e2e 2>&1 | grep '^{')" >> gpurun_out/cl4_step.log
  done
fi
