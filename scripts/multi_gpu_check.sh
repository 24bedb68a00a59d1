#!/bin/bash
# Multi-GPU round check (under gpurun --gpus 4): parity tests at P = 2/4, the three
# strategies at N = 4, peer-copy mechanism comparison, N = 2 bench.
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_step.py -x -q -k "two or four" 2>&1 | tail -4
N=4 bash scripts/strategies.sh
BM_PEER_COPY=sm timeout 600 $TR --nproc-per-node 4 --master-port 29781 bench.py --gpus 4 --steps 5 --warmup 3 --no-e2e \
  > gpurun_out/bench_n4_cecopy.log 2>&1
grep '^{' gpurun_out/bench_n4_cecopy.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bigmac SM-copy samples/s %.2f ms %.1f' % (d['value'], d['ms_per_step']))"
timeout 600 $TR --nproc-per-node 2 --master-port 29782 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/bench_n2_v5.log 2>&1
grep '^{' gpurun_out/bench_n2_v5.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N=2 samples/s %.2f ms %.1f' % (d['value'], d['ms_per_step']))"
