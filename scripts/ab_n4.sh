#!/bin/bash
# 4-GPU A/B of bench variants, alternating, one JSON summary line per run
run() {  # label, extra args
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29621 \
    bench.py --gpus 4 --steps 10 --warmup 3 --no-extra --no-cpu --no-e2e $2 > gpurun_out/ab_n4.log 2>&1
  python - "$1" <<'PY'
import json, sys
l = [x for x in open("gpurun_out/ab_n4.log") if x.startswith("{")]
if not l:
    print(sys.argv[1], "FAILED"); sys.exit(0)
d = json.loads(l[-1])
print(json.dumps({"variant": sys.argv[1], "value": round(d["value"], 2), "ms": round(d["ms_per_step"], 1),
                  "bubble": [round(x, 3) for x in d["bubble"]["per_rank"]], "gen_exclude": d["config"]["gen_exclude"],
                  "fsdp": d["fsdp"], "clock": d["clocks"]["sm_mhz"] if d["clocks"] else None}))
PY
}
for i in 1 2; do
  run "genx-auto" "--gen-exclude auto"
  run "genx-none" "--gen-exclude none"
done
run "fsdp-pull" "--fsdp pull --gen-exclude none"
run "fsdp-allgather" "--fsdp allgather --gen-exclude none"
run "fsdp-off" "--gen-exclude none"
