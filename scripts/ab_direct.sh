# SwiGLU-backward epilogue: direct register stores vs smem staging + TMA stores
export CUDA_DEVICE_MAX_CONNECTIONS=32
BM_DSWIGLU_DIRECT=1 timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "swiglu" > gpurun_out/direct_tests.log 2>&1
tail -1 gpurun_out/direct_tests.log
BM_DSWIGLU_DIRECT=1 timeout 900 python -m pytest tests/test_gpu_step.py -q -x -k "single_gpu and bf16" > gpurun_out/direct_step_tests.log 2>&1
tail -1 gpurun_out/direct_step_tests.log
for v in 0 1 0 1; do
  echo "== DIRECT=$v" >> gpurun_out/direct_knob.log
  BM_DSWIGLU_DIRECT=$v timeout 600 python scripts/gemm_ab_knob.py 2 bk128 2>&1 | grep dswiglu >> gpurun_out/direct_knob.log
done
for v in 0 1 0 1; do
  echo "DIRECT=$v $(BM_DSWIGLU_DIRECT=$v timeout 300 python bench.py --steps 6 --warmup 3 --no-extra --sweep '' --no-cpu --no-e2e 2>&1 | grep '^{')" >> gpurun_out/direct_step.log
done
