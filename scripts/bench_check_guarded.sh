export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 900 python bench.py > gpurun_out/bench_n1_guarded.log 2>&1
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29702 bench.py --gpus 2 > gpurun_out/bench_n2_guarded.log 2>&1
for f in gpurun_out/bench_n1_guarded.log gpurun_out/bench_n2_guarded.log; do python -c "
import json,sys
for l in open('$f'):
    if l.startswith('{'):
        d=json.loads(l); print('$f', d['value'], [k for k in d if isinstance(d[k], dict) and 'error' in d[k]], sorted(k for k in ('c4_single_gpu','batch_sweep','c2_m16_per_replica','zb_h1','c4_strong') if k in d))
"; done
