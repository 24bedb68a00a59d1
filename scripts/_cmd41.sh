TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 4"
for R in 0 8 16 32; do
  BM_GEN_RESERVE_SMS=$R timeout 400 $TR --master-port $((29700 + R)) bench.py --gpus 4 --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_n4_res$R.log 2>&1
  grep '^{' gpurun_out/bench_n4_res$R.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('reserve $R samples/s %.2f ms %.1f' % (d['value'], d['ms_per_step']))"
done
BM_GEN_RESERVE_SMS=16 timeout 300 $TR --master-port 29861 scripts/trace_step.py --config C2 --M 16 --strategy bigmac --out gpurun_out/trace_c2_n4_bigmac_res16.json 2>&1 | grep '^{' > gpurun_out/trace_c2_n4_bigmac_res16.summary.json
