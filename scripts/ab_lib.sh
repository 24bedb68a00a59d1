# A/B of two library builds (paper_2605_25451_b200/libbigmac_old.so vs libbigmac_new.so): parity, GEMM shapes, C2 step
export CUDA_DEVICE_MAX_CONNECTIONS=32
D=paper_2605_25451_b200
cp $D/libbigmac_new.so $D/libbigmac.so
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_step.py -q -x -k "not multirank and not timeout" > gpurun_out/lib_tests.log 2>&1; tail -1 gpurun_out/lib_tests.log
timeout 600 python scripts/gemm_ab.py $D/libbigmac_old.so $D/libbigmac_new.so > gpurun_out/lib_gemm_ab.log 2>&1
for r in 1 2; do for v in old new; do
  cp $D/libbigmac_$v.so $D/libbigmac.so
  echo "$v $(timeout 300 python bench.py --steps 6 --warmup 3 --no-extra --sweep '' --no-cpu --no-e2e 2>&1 | grep '^{')" >> gpurun_out/lib_step.log
done; done
cp $D/libbigmac_new.so $D/libbigmac.so
