# 256x512 vs 256x256 CTA-pair tiles: parity tests, gemm_bench under each setting, C2 step A/B
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "bn512 or pairs or epilogues or fused_swiglu" > gpurun_out/bn512_tests.log 2>&1
tail -3 gpurun_out/bn512_tests.log
for v in 0 1 2; do
  echo "== BM_GEMM_BN512=$v" >> gpurun_out/bn512_bench.log
  BM_GEMM_BN512=$v timeout 300 python scripts/gemm_bench.py >> gpurun_out/bn512_bench.log 2>&1
done
for v in 0 2 0 2; do
  echo "BN512=$v $(BM_GEMM_BN512=$v timeout 300 python bench.py --steps 6 --warmup 3 --no-extra --sweep '' --no-cpu --no-e2e 2>&1 | grep '^{')" >> gpurun_out/bn512_step.log
done
