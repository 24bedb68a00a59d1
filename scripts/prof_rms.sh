export CUDA_DEVICE_MAX_CONNECTIONS=32
for i in 1 2; do python scripts/prof_elementwise.py 2>&1 | grep -i rmsnorm >> gpurun_out/rms_prof.log; done
for i in 1 2; do echo "$(timeout 300 python bench.py --steps 6 --warmup 3 --no-extra --sweep '' --no-cpu --no-e2e 2>&1 | grep '^{')" >> gpurun_out/rms_step.log; done
