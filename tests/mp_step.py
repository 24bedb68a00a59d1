"""One rank of a multi-GPU parity run (launched by tests/test_gpu_step.py via torchrun).

usage: mp_step.py CONFIG P M V DTYPE GEN_PLACE[+head_dp][+last<n>] [D]
D > 1: D pipeline replicas of P stages (world = P D); replica k runs microbatches
[kM, (k+1)M) of one global batch of M D microbatches, and every gradient is
compared with the oracle's gradient of that global batch.
Every rank runs bm_step on its own GPU; rank 0 gathers all gradients and
compares them with the fp64 oracle (normwise rel tol 1e-4 fp32 / 2e-2 bf16).
"""
import os

# one hardware work queue per stream (compute, P-1 comm, generator, NCCL): a comm
# stream parked on a credit wait must not block unrelated streams sharing its queue
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from synth import edge_counts, edge_shape, get_config, make_batch, make_weights, slice_batch  # noqa: E402


def main():
    name, P, M, V, dtype, gen = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), sys.argv[5], sys.argv[6]
    D = int(sys.argv[7]) if len(sys.argv) > 7 else 1
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    assert world == P * D, (world, P, D)
    # BM_TEST_ONE_GPU=1: every rank on cuda:0 (the single-GPU multi-rank fixture: CUDA
    # IPC works between processes of one device; the step-end sums then run over peer
    # memory, bm_ctx_init_peer_sum, because NCCL rejects duplicate devices)
    one_gpu = os.environ.get("BM_TEST_ONE_GPU") == "1"
    torch.cuda.set_device(0 if one_gpu else int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("gloo")
    from paper_2605_25451_b200.runtime import Runtime
    edge = "edge" in gen.split("+")
    gen = "+".join(t for t in gen.split("+") if t != "edge")
    cfg = get_config(name, P=P, M=M, V=V)
    cfg_global = get_config(name, P=P, M=M * D, V=V)
    if edge:   # degenerate row counts (synth.edge_counts), buffers sized for [0, S]
        cfg, cfg_global = edge_shape(cfg), edge_shape(cfg_global)
        n_mod, n_gen = edge_counts(cfg_global, M * D)
        W, B_global = make_weights(cfg), make_batch(cfg_global, n_mod=n_mod, n_gen=n_gen)
    else:
        W, B_global = make_weights(cfg), make_batch(cfg_global)
    replica = rank // P
    B = slice_batch(B_global, replica * M, (replica + 1) * M)
    # strategy spec: "<gen_place>", "entry_stage+<gen_place>" (memory-efficient baseline),
    # "ce" (compute-efficient baseline: all encoder forwards first, W = M / P);
    # "<gen_place>+head_dp": the LM head + CE DP-sharded with the generator (BM_HEAD_DP_SHARD)
    # "...+last<n>": last_stage_layers = n (uneven LLM layer partition, bigmac.h)
    # "...+split<a>-<b>-...": explicit stage_layers
    head, last, split = "auto", 0, None
    toks = gen.split("+")
    for t in toks:
        if t.startswith("split"):
            split = [int(x) for x in t[5:].split("-")]
    toks = [t for t in toks if not t.startswith("split")]
    if "head_dp" in toks:
        head = "dp_shard"
    for t in toks:
        if t.startswith("last") and t[4:].isdigit():
            last = int(t[4:])
    gen = "+".join(t for t in toks if t != "head_dp" and not (t.startswith("last") and t[4:].isdigit()))
    if gen == "ce":
        kw = {"warmup_units": M // P}
    elif gen.startswith("entry_stage+"):
        kw = {"enc_place": "entry_stage", "gen_place": gen.split("+")[1]}
    else:
        kw = {"gen_place": gen}
    rt = Runtime(cfg, dtype, rank=rank, world=world, sched_kw=kw, head_place=head, last_stage_layers=last,
                 stage_layers=split)
    rt.load_weights(W)
    db = rt.device_batch(B)
    for _ in range(2):
        rt.step(db)
    torch.cuda.synchronize()
    loss, ce, mse = rt.losses()
    grads = {n: rt.grad(n) for n in rt.names()}
    kinds = {n: rt.params[n][4] for n in rt.names()}
    allg = [None] * world
    dist.gather_object((grads, kinds, loss, ce, mse), allg if rank == 0 else None, dst=0)
    if rank == 0:
        from oracle import model as om
        loss_ref, per_ref, G_ref = om.step_fp64(cfg_global, W, B_global)
        tol = 1e-4 if dtype == "f32" else 2e-2
        ok = True
        for r, (g, k, l_, c_, m_) in enumerate(allg):
            if abs(l_ - loss_ref) > tol * abs(loss_ref):
                print(f"rank {r} loss {l_} vs {loss_ref}")
                ok = False
            q = r // P   # replica: its own microbatches' loss terms
            ce_ref = np.array([x for x, _ in per_ref[q * M:(q + 1) * M]])
            mse_ref = np.array([y for _, y in per_ref[q * M:(q + 1) * M]])
            if (np.linalg.norm(c_ - ce_ref) > tol * np.linalg.norm(ce_ref) or
                    np.linalg.norm(m_ - mse_ref) > tol * max(np.linalg.norm(mse_ref), 1e-30)):
                print(f"rank {r} per-microbatch loss terms differ")
                ok = False
            for n, v in g.items():
                ref = G_ref[n]
                e = np.linalg.norm(v - ref) / max(np.linalg.norm(ref), 1e-30)
                if e > tol:
                    print(f"rank {r} grad {n} rel err {e:.3e}")
                    ok = False
        seen = set()
        for g, _, _, _, _ in allg:
            seen |= set(g)
        missing = set(G_ref) - seen
        if missing:
            print("missing grads", missing)
            ok = False
        print("PARITY OK" if ok else "PARITY FAIL", loss, loss_ref, "sum_mode", rt.sum_mode)
    dist.barrier()
    rt.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
