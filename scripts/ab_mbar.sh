# CTA-scope barrier polls (no CCTL.IVALL per poll) vs cluster scope: GEMM shapes and the C2 step
export CUDA_DEVICE_MAX_CONNECTIONS=32
for v in cluster cta cluster cta; do
  echo "== $v" >> gpurun_out/mbar_gemm.log
  BM_MBAR_SCOPE=$v timeout 600 python scripts/gemm_bench.py 2>&1 | grep -E "C2 |dswiglu" | head -9 >> gpurun_out/mbar_gemm.log
done
for v in cluster cta cluster cta; do
  echo "$v $(BM_MBAR_SCOPE=$v timeout 300 python bench.py --steps 6 --warmup 3 --no-extra --sweep '' --no-cpu --no-e2e 2>&1 | grep '^{')" >> gpurun_out/mbar_step.log
done
