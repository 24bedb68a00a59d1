# raster group G of the pair GEMM with 128-deep K blocks: standalone and C2 step
export CUDA_DEVICE_MAX_CONNECTIONS=32
for g in 8 4 16 8 4 16; do
  echo "== G=$g" >> gpurun_out/group_gemm.log
  BM_GEMM_GROUP=$g timeout 300 python scripts/gemm_bench.py 2>&1 | grep -E '"C2 |"C4 ' >> gpurun_out/group_gemm.log
done
for g in 8 4 16 8 4 16; do
  echo "G=$g $(BM_GEMM_GROUP=$g timeout 300 python bench.py --steps 6 --warmup 3 --no-extra --sweep '' --no-cpu --no-e2e 2>&1 | grep '^{')" >> gpurun_out/group_step.log
done
