# kernel names + key counters of our pair GEMM and cuBLAS on the C2 LLM shapes (one replay each)
export CUDA_DEVICE_MAX_CONNECTIONS=32
ncu --clock-control none -k regex:'gemm2_kernel|nvjet|cutlass|sm100|xmma|gemm' \
  --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,launch__grid_size,launch__cluster_dim_x,launch__cluster_dim_y,l1tex__m_xbar2l1tex_read_bytes.sum,lts__t_sectors_srcunit_ltcfabric.sum,sm__cycles_elapsed.avg.per_second,launch__shared_mem_per_block_dynamic,dram__bytes_read.sum \
  --csv python scripts/ncu_gemm_vs_cublas.py c2 > gpurun_out/ncu_gvc_c2.csv 2> gpurun_out/ncu_gvc_c2.err
