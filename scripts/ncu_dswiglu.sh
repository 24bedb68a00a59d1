export CUDA_DEVICE_MAX_CONNECTIONS=32
python scripts/ncu_dswiglu.py && ncu --set full --import-source on --clock-control none -k regex:gemm2 -s 1 -c 1 \
  -o gpurun_out/prof_dswiglu python scripts/ncu_dswiglu.py > gpurun_out/ncu_dswiglu.log 2>&1
