# pipelined wide RMSNorm backward: parity (both settings), standalone and C2 step A/B
export CUDA_DEVICE_MAX_CONNECTIONS=32
for v in 1 0; do BM_RMS_PIPE=$v timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k rmsnorm 2>&1 | tail -1; done
BM_RMS_PIPE=1 timeout 600 python -m pytest tests/test_gpu_step.py -q -x -k "single_gpu and not medium" 2>&1 | tail -1
for v in 0 1 0 1; do echo "PIPE=$v $(BM_RMS_PIPE=$v python scripts/prof_elementwise.py 2>&1 | grep 'rmsnorm_bwd')" >> gpurun_out/rmspipe_prof.log; done
for v in 0 1 0 1; do
  echo "PIPE=$v $(BM_RMS_PIPE=$v timeout 300 python bench.py --steps 6 --warmup 3 --no-extra --sweep '' --no-cpu --no-e2e 2>&1 | grep '^{')" >> gpurun_out/rmspipe_step.log
done
