# full GPU suite + smoke + default bench (N = 1) of HEAD on one B200
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_full.log 2>&1
tail -3 gpurun_out/pytest_gpu_full.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_n1_full.log 2>&1; tail -c 600 gpurun_out/bench_n1_full.log
