"""Per-op trace of one nested-pipeline step on every rank -> Chrome trace JSON.

    python -m torch.distributed.run --nproc-per-node P scripts/trace_step.py [--config C2] [--M 16]
        [--strategy bigmac|compute_efficient|memory_efficient] [--out profiles/r01/trace.json]

Each rank records CUDA events around every op (compute ops on the compute /
generator stream, the NVLink copy of every send on its comm stream, the moment
every receive's flag wait is satisfied); rank 0 writes one Chrome-trace file
(pid = rank, tid = stream) and prints a per-rank summary: busy time per stream
and the compute-stream idle gaps, attributed to the op that followed them.
"""
import argparse
import json
import os

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")   # before the CUDA context (executor.cu)
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

STREAMS = {0: "compute", 1: "generator"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--M", type=int, default=16)
    ap.add_argument("--V", type=int, default=1)
    ap.add_argument("--strategy", default="bigmac")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--head", default="auto", choices=["auto", "last_stage", "dp_shard"])
    ap.add_argument("--last-stage-layers", type=int, default=0)
    ap.add_argument("--stage-layers", default="", help="explicit LLM layers per stage, e.g. 4,4,5,3")
    ap.add_argument("--halves", action="store_true", help="--stage-layers in half-layer units (stage_halves)")
    ap.add_argument("--gen-exclude", type=int, default=0, help="bit mask (bigmac.h gen_exclude)")
    ap.add_argument("--enc-exclude", type=int, default=0, help="bit mask (bm_sched_cfg.enc_exclude)")
    ap.add_argument("--llm-sched", default="auto", choices=["auto", "zb_h1"])
    ap.add_argument("--out", default="gpurun_out/trace.json")
    a = ap.parse_args()
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    group = None
    if world > 1:
        dist.init_process_group("cpu:gloo,cuda:nccl", device_id=torch.device("cuda", int(os.environ.get("LOCAL_RANK", rank))))
        group = dist.new_group(backend="gloo")
    from synth import get_config, make_batch
    from paper_2605_25451_b200.runtime import Runtime
    cfg = get_config(a.config, P=world, M=a.M, V=a.V)
    if a.llm_sched == "zb_h1":
        cfg = cfg.replace(llm_sched="zb_h1")
    kw = {"bigmac": {}, "compute_efficient": {"warmup_units": cfg.M // world},
          "memory_efficient": {"enc_place": "entry_stage", "gen_place": "last_stage"}}[a.strategy]
    kw = dict(kw, llm_sched=cfg.llm_sched)
    if a.enc_exclude:
        kw["enc_exclude"] = a.enc_exclude
    rt = Runtime(cfg, "bf16", rank=rank, world=world, group=group, sched_kw=kw, head_place=a.head,
                 last_stage_layers=a.last_stage_layers,
                 stage_layers=[int(v) for v in a.stage_layers.split(",")] if a.stage_layers else None,
                 gen_exclude=a.gen_exclude, stage_halves=a.halves)
    rt.init_random_weights(1)
    db = rt.device_batch(make_batch(cfg))
    for _ in range(a.warmup):
        rt.step(db)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier(group=group)
    rt.set_trace(True)
    rt.step(db)
    torch.cuda.synchronize()
    tr = rt.trace()
    rt.set_trace(False)
    allt = [None] * world
    if world > 1:
        dist.gather_object(tr, allt if rank == 0 else None, dst=0, group=group)
    else:
        allt = [tr]
    if rank == 0:
        events = []
        for r, recs in enumerate(allt):
            for x in recs:
                tid = STREAMS.get(x["stream"], "encoder" if x["stream"] == 2 + world else f"comm->{x['stream'] - 2}")
                name = x["kind"] if x["mb"] < 0 else f"{x['kind']} mb{x['mb']}"
                dur = max(x["t1"] - x["t0"], 0.001)
                events.append({"name": name, "ph": "X", "pid": f"rank {r}", "tid": tid,
                               "ts": x["t0"] * 1e3, "dur": dur * 1e3, "args": {"op": x["op"]}})
        os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
        with open(a.out, "w") as f:
            json.dump({"traceEvents": events, "displayTimeUnit": "ms"}, f)
        summ = []
        for r, recs in enumerate(allt):
            comp = sorted([x for x in recs if x["stream"] in (0, 1, 2 + world) and x["kind"] not in ("Recv",)],
                          key=lambda x: x["t0"])
            main = [x for x in comp if x["stream"] == 0]
            end = max(x["t1"] for x in recs)
            busy = {}
            for x in recs:
                if x["kind"] == "Recv":
                    continue
                k = STREAMS.get(x["stream"], "encoder" if x["stream"] == 2 + world else "comm")
                busy[k] = busy.get(k, 0.0) + (x["t1"] - x["t0"])
            gaps = []
            prev = 0.0
            for x in main:
                if x["t0"] - prev > 0.05:
                    gaps.append((x["t0"] - prev, x["kind"], x["mb"], x["op"]))
                prev = max(prev, x["t1"])
            gaps.sort(reverse=True)
            per_kind, n_kind = {}, {}
            for x in comp:
                per_kind[x["kind"]] = per_kind.get(x["kind"], 0.0) + x["t1"] - x["t0"]
                n_kind[x["kind"]] = n_kind.get(x["kind"], 0) + 1
            idle_by_next = {}
            for g in gaps:
                idle_by_next[g[1]] = idle_by_next.get(g[1], 0.0) + g[0]
            # compute-stream idle as a fraction of the step vs the 1F1B closed form
            # (P-1)/(MV+P-1): the measured idle also holds stage imbalance
            summ.append({"rank": r, "step_ms": end, "busy_ms": busy,
                         "compute_idle_frac": sum(g[0] for g in gaps) / end if end > 0 else None,
                         "bubble_bound_1f1b": (world - 1) / (a.M * a.V + world - 1),
                         "compute_idle_ms": sum(g[0] for g in gaps),
                         "op_ms_by_kind": per_kind,
                         "op_mean_ms": {k: per_kind[k] / n_kind[k] for k in per_kind},
                         "compute_idle_ms_by_next_op": idle_by_next,
                         "top_idle_gaps_before": [{"ms": round(g[0], 3), "op": g[1], "mb": g[2], "idx": g[3]}
                                                  for g in gaps[:8]]})
        print(json.dumps({"config": a.config, "P": world, "M": a.M, "strategy": a.strategy, "head": a.head,
                          "ranks": summ}))
    if world > 1:
        dist.barrier(group=group)
    rt.close()


if __name__ == "__main__":
    main()
