# C2 step and C4 (M = 8 at P = 1) A/B of the pair-tile policy: 256x256 only vs the cost model
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "bn512" > gpurun_out/bn512_tests.log 2>&1
tail -1 gpurun_out/bn512_tests.log
for v in 0 2 0 2; do
  echo "BN512=$v $(BM_GEMM_BN512=$v timeout 300 python bench.py --steps 6 --warmup 3 --no-extra --sweep '' --no-cpu --no-e2e 2>&1 | grep '^{')" >> gpurun_out/bn512_step2.log
done
for v in 0 2; do
  echo "BN512=$v $(BM_GEMM_BN512=$v timeout 600 python bench.py --config C4 --microbatches 8 --steps 3 --warmup 3 --no-extra --sweep '' --no-cpu --no-e2e 2>&1 | grep '^{')" >> gpurun_out/bn512_step2.log
done
