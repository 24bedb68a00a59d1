"""C5: global-batch sweep -- peak HBM per GPU and samples/s vs M at fixed P.

    python -m torch.distributed.run --nproc-per-node P scripts/c5_sweep.py [--config C2] [--ms 8,16,...]

For every M the schedule's stash plan (W encoder units, peak in-flight LLM
microbatches, one generator shard) is independent of M, so peak HBM must stay
flat for M >= P (the O(1) encoder/generator memory claim).
Prints one JSON line per M on rank 0.
"""
import argparse
import json
import os

# one hardware work queue per stream (compute, P-1 comm, generator, NCCL): a comm
# stream parked on a credit wait must not block unrelated streams sharing its queue
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--ms", default="8,16,32,64,128,256")
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--strategy", default="bigmac", choices=["bigmac", "compute_efficient", "memory_efficient"])
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    group = None
    if world > 1:
        dist.init_process_group("cpu:gloo,cuda:nccl", device_id=torch.device("cuda", local))
        group = dist.new_group(backend="gloo")
    from synth import get_config, make_batch
    from paper_2605_25451_b200.runtime import Runtime
    for M in [int(x) for x in args.ms.split(",")]:
        if M % world:
            continue
        cfg = get_config(args.config, P=world, M=M, V=1)
        torch.cuda.empty_cache()
        torch.cuda.reset_peak_memory_stats()
        kw = {"bigmac": {}, "compute_efficient": {"warmup_units": M // world},
              "memory_efficient": {"enc_place": "entry_stage", "gen_place": "last_stage"}}[args.strategy]
        rt = Runtime(cfg, "bf16", rank=rank, world=world, group=group, sched_kw=kw)
        rt.init_random_weights(1)
        mem0 = torch.cuda.memory_allocated()
        db = rt.device_batch(make_batch(cfg))
        batch_bytes = torch.cuda.memory_allocated() - mem0   # resident inputs (grow with M)
        rt.step(db)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if world > 1:
            dist.barrier(group=group)
        e0.record()
        for _ in range(args.steps):
            rt.step(db)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.steps
        peak = torch.cuda.max_memory_allocated() / 1e9
        st = rt.sched.stats(rank)
        t = torch.tensor([ms, peak], dtype=torch.float64)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
        stash = rt.stash_peak()
        if rank == 0:
            print(json.dumps({"config": args.config, "strategy": args.strategy, "P": world, "M": M, "global_batch": M,
                              "work_bytes_rank0": rt.sizes.work_bytes, "input_batch_bytes_rank0": batch_bytes,
                              "samples_per_s": M / (t[0].item() / 1e3), "ms_per_step": t[0].item(),
                              "peak_hbm_gb_per_gpu_max": t[1].item(),
                              "rank0_stash_bytes_enc_llm_gen": stash,
                              "rank0_peak_enc_units": st.peak_enc_units, "rank0_peak_llm_inflight": st.peak_llm_inflight,
                              "rank0_peak_gen_shards": st.peak_gen_shards}), flush=True)
        rt.close()
        del rt, db
        if world > 1:
            dist.barrier(group=group)


if __name__ == "__main__":
    main()
