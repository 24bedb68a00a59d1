#!/bin/bash
# BigMac vs the paper's two baselines on the same executor (C2 model), P = N GPUs.
# usage (under gpurun --gpus N): N=4 bash scripts/strategies.sh
mkdir -p gpurun_out
N=${N:-4}
for S in bigmac compute_efficient memory_efficient; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
      --master-port $((29700 + RANDOM % 100)) bench.py --gpus $N --steps 5 --warmup 3 --no-e2e --strategy $S \
      > gpurun_out/strat_${S}_n$N.log 2>&1
  grep '^{' gpurun_out/strat_${S}_n$N.log | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$S', 'samples/s %.2f' % d['value'], 'ms/step %.1f' % d['ms_per_step'], 'peak HBM/GPU %.2f GB' % d['peak_hbm_gb_per_gpu'],
      'rank0 stash enc/llm/gen', d['stash_peak_bytes_rank0'])"
done
