#!/bin/bash
# bench.py at N = 1, 2, 4 on one box (run under gpurun --gpus 4)
mkdir -p gpurun_out
STEPS=${STEPS:-10}
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --steps $STEPS --warmup 3 > gpurun_out/bench_n1.log 2>&1
for N in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
      --master-port $((29600 + N)) bench.py --gpus $N --steps $STEPS --warmup 3 > gpurun_out/bench_n$N.log 2>&1
done
for N in 1 2 4; do echo "== N=$N"; grep '^{' gpurun_out/bench_n$N.log | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print({k:d.get(k) for k in ['value','ms_per_step','gpu_launches','peak_hbm_gb_per_gpu']}, 'roof', d['roofline']['achieved'], d['roofline']['frac'], d['roofline']['gemm_share_of_step'], 'step', d['step_roofline']['frac'], 'e2e', (d.get('e2e') or {}).get('value'), d.get('clocks'))
"; tail -3 gpurun_out/bench_n$N.log | cut -c1-300; done
