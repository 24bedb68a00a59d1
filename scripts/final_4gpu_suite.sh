# the whole GPU suite on a 4-GPU box (multi-rank cases one GPU per rank over NCCL)
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 3000 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_4gpu_final.log 2>&1
tail -3 gpurun_out/pytest_gpu_4gpu_final.log
