# N = 4, C2, halves + ZB-H1: where the encoder / generator run, SM reserve for the generator stream
export CUDA_DEVICE_MAX_CONNECTIONS=32
run() { timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 \
  --master-port $1 bench.py --gpus 4 --steps 6 --warmup 3 --no-extra --sweep '' --no-cpu --no-e2e --partition halves --llm-sched zb_h1 $2 2>&1 | grep '^{' ; }
echo "auto $(run 29610 '')" >> gpurun_out/ab_place_n4.log
echo "x012 $(run 29620 '--gen-exclude 0,1,2 --enc-exclude 0,1,2')" >> gpurun_out/ab_place_n4.log
echo "g012_e02 $(run 29630 '--gen-exclude 0,1,2 --enc-exclude 0,2')" >> gpurun_out/ab_place_n4.log
echo "u9_9_8_6 $(run 29640 '--stage-layers 9,9,8,6 --gen-exclude 0,1 --enc-exclude 0,1')" >> gpurun_out/ab_place_n4.log
echo "auto_res8 $(BM_GEN_RESERVE_SMS=8 run 29650 '')" >> gpurun_out/ab_place_n4.log
echo "x012 $(run 29660 '--gen-exclude 0,1,2 --enc-exclude 0,1,2')" >> gpurun_out/ab_place_n4.log
echo "auto $(run 29670 '')" >> gpurun_out/ab_place_n4.log
