export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 3000 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_final2.log 2>&1
tail -2 gpurun_out/pytest_gpu_final2.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final2.log 2>&1; tail -1 gpurun_out/smoke_final2.log
timeout 900 python bench.py > gpurun_out/bench_n1_final2.log 2>&1
