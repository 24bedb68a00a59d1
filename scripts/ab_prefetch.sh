# epilogue L2 prefetch A/B: GEMM knob bench (env per process) and C2 step
export CUDA_DEVICE_MAX_CONNECTIONS=32
for v in 0 1 0 1; do
  echo "== BM_EPI_PREFETCH=$v" >> gpurun_out/pf_gemm.log
  BM_EPI_PREFETCH=$v timeout 300 python scripts/gemm_ab_knob.py 2 2>&1 | grep -E "dswiglu|fwd\\+res" >> gpurun_out/pf_gemm.log
done
for v in 0 1 0 1; do
  echo "PF=$v $(BM_EPI_PREFETCH=$v timeout 300 python bench.py --steps 6 --warmup 3 --no-extra --sweep '' --no-cpu --no-e2e 2>&1 | grep '^{')" >> gpurun_out/pf_step.log
done
