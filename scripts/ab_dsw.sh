# SwiGLU-backward GEMM smem variants: parity then A/B (standalone and C2 step)
export CUDA_DEVICE_MAX_CONNECTIONS=32
for v in 1 2; do
  BM_DSW_VARIANT=$v timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "dswiglu or fused_swiglu" > gpurun_out/dsw_tests_$v.log 2>&1
  tail -1 gpurun_out/dsw_tests_$v.log
done
for r in 1 2; do for v in 0 1 2; do
  echo "== VAR=$v" >> gpurun_out/dsw_knob.log
  BM_DSW_VARIANT=$v timeout 600 python scripts/gemm_ab_knob.py 2 bk128 2>&1 | grep dswiglu >> gpurun_out/dsw_knob.log
done; done
for r in 1 2; do for v in 0 1 2; do
  echo "VAR=$v $(BM_DSW_VARIANT=$v timeout 300 python bench.py --steps 6 --warmup 3 --no-extra --sweep '' --no-cpu --no-e2e 2>&1 | grep '^{')" >> gpurun_out/dsw_step.log
done; done
