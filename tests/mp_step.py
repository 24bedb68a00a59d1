"""Ranks of a multi-rank parity run (launched by tests/test_gpu_step.py via torchrun).

usage: mp_step.py CASE [CASE ...]
  CASE = CONFIG:P:M:V:DTYPE:SPEC:D[:FLAGS]   (FLAGS comma-separated: peer, gm2, es)
Every case runs in the same processes, one after the other (one process start
and CUDA context per rank for the whole batch).  world = P D for every case.
D > 1: D pipeline replicas of P stages; replica k runs microbatches [kM, (k+1)M)
of one global batch of M D microbatches, and every gradient is compared with the
oracle's gradient of that global batch.  Rank 0 gathers all gradients and
compares them with the fp64 oracle (normwise rel tol 1e-4 fp32 / 2e-2 bf16),
printing one line "CASE <case> PARITY OK|FAIL ..." per case.
SPEC: "<gen_place>", "entry_stage+<gen_place>" (memory-efficient baseline), "ce"
(compute-efficient baseline: all encoder forwards first, W = M / P); modifiers
"+head_dp" (LM head + CE DP-sharded with the generator), "+last<n>"
(last_stage_layers = n), "+split<a>-<b>-..." (explicit stage_layers), "+edge"
(degenerate row counts, synth.edge_counts), "+fsdp" / "+fsdpag" (FSDP with the
one-sided pull / the all-gather baseline), "+genx<mask>" (ranks in the bit mask take
no generator rows), "+encx<mask>" (ranks in the mask run no encoder microbatch),
"+zb" (ZB-H1 zero-bubble LLM schedule, B/W split, reading R23), "+halves<a>-<b>-..."
(explicit partition in half-layer units, stage boundaries inside layers, reading R24).
FLAGS: peer = force the library's peer-memory step-end sum (BM_STEP_SUM=peer);
gm2 = every bf16 contraction on the CTA-pair GEMM (bm_k_gemm_mode 2); es = encoder ops on
their own stream (bm_model_cfg.enc_stream = 1).
"""
import os

# one hardware work queue per stream (compute, P-1 comm, generator, NCCL): a comm
# stream parked on a credit wait must not block unrelated streams sharing its queue
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import sys
import time
import traceback

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from synth import edge_counts, edge_shape, get_config, make_batch, make_weights, slice_batch  # noqa: E402


def parse_spec(spec, M, P):
    head, last, split = "auto", 0, None
    toks = spec.split("+")
    edge = "edge" in toks
    fsdp = "pull" if "fsdp" in toks else ("allgather" if "fsdpag" in toks else "off")
    genx = sum(int(t[4:]) for t in toks if t.startswith("genx"))
    encx = sum(int(t[4:]) for t in toks if t.startswith("encx"))
    zb = "zb" in toks
    toks = [t for t in toks if t not in ("edge", "fsdp", "fsdpag", "zb") and not t.startswith(("genx", "encx"))]
    halves = False
    for t in toks:
        if t.startswith("split"):
            split = [int(x) for x in t[5:].split("-")]
        if t.startswith("halves"):   # explicit partition in half-layer units (stage_halves, R24)
            split, halves = [int(x) for x in t[6:].split("-")], True
    toks = [t for t in toks if not t.startswith(("split", "halves"))]
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
    if encx:
        kw["enc_exclude"] = encx
    if zb:
        kw["llm_sched"] = "zb_h1"
    return kw, head, last, split, edge, fsdp, genx, halves


def run_case(case, rank, world):
    from paper_2605_25451_b200 import _lib as L
    from paper_2605_25451_b200.runtime import Runtime
    parts = case.split(":")
    name, P, M, V, dtype, spec, D = parts[0], int(parts[1]), int(parts[2]), int(parts[3]), parts[4], parts[5], int(parts[6])
    flags = parts[7].split(",") if len(parts) > 7 and parts[7] else []
    assert world == P * D, (case, world)
    kw, head, last, split, edge, fsdp, genx, halves = parse_spec(spec, M, P)
    cfg = get_config(name, P=P, M=M, V=V)
    cfg_global = get_config(name, P=P, M=M * D, V=V)
    if edge:   # degenerate row counts, buffers sized for [0, S]
        cfg, cfg_global = edge_shape(cfg), edge_shape(cfg_global)
        n_mod, n_gen = edge_counts(cfg_global, M * D)
        W, B_global = make_weights(cfg), make_batch(cfg_global, n_mod=n_mod, n_gen=n_gen)
    else:
        W, B_global = make_weights(cfg), make_batch(cfg_global)
    replica = rank // P
    B = slice_batch(B_global, replica * M, (replica + 1) * M)
    os.environ["BM_STEP_SUM"] = "peer" if "peer" in flags else "auto"
    L.call("bm_k_gemm_mode", 2 if "gm2" in flags else 0)
    rt = Runtime(cfg, dtype, rank=rank, world=world, sched_kw=kw, head_place=head, last_stage_layers=last,
                 stage_layers=split, fsdp=fsdp, gen_exclude=genx, stage_halves=halves,
                 enc_stream=1 if "es" in flags else 0)
    rt.load_weights(W)
    db = rt.device_batch(B)
    for _ in range(2):
        rt.step(db)
    rt.step_wait(300.0)   # a hang becomes BM_E_TIMEOUT naming the blocked op
    torch.cuda.synchronize()
    loss, ce, mse = rt.losses()
    grads = {n: rt.grad(n) for n in rt.names()}
    meta = {"params": dict(rt.params), "shard": (rt.dp_lo, rt.dp_hi), "w_elems": rt.w_elems,
            "total": rt.total_elems, "pull": rt.pull_bytes()}
    allg = [None] * world
    dist.gather_object((grads, loss, ce, mse, meta), allg if rank == 0 else None, dst=0)
    if rank == 0:
        from oracle import model as om
        loss_ref, per_ref, G_ref = om.step_fp64(cfg_global, W, B_global)
        tol = 1e-4 if dtype == "f32" else 2e-2
        msgs = []
        if fsdp != "off":
            # FSDP: rank r's DP gradients are valid on its shard [lo_r, hi_r) of the DP
            # elements only (reduce-scatter); stitch the shards into full DP gradients
            stitched = {}
            for g, _, _, _, meta in allg:
                lo, hi = meta["shard"]
                for n, (rows, cols, ld, off, kind) in meta["params"].items():
                    if kind != 0:
                        continue
                    e = off + np.arange(rows)[:, None] * ld + np.arange(cols)[None, :]
                    own = ((e >= lo) & (e < hi)).reshape(g[n].shape)
                    tgt = stitched.setdefault(n, np.full(g[n].shape, np.nan))
                    tgt[own] = g[n][own]
            for g, _, _, _, meta in allg:
                for n in stitched:
                    g[n] = stitched[n]
                if P > 1 and not meta["w_elems"] < meta["total"]:
                    msgs.append("FSDP weights buffer is not sharded")
            if P > 1 and not any(meta["pull"] > 0 for *_, meta in allg):
                msgs.append("FSDP pulled no bytes from peers")
        for r, (g, l_, c_, m_, _) in enumerate(allg):
            if abs(l_ - loss_ref) > tol * abs(loss_ref):
                msgs.append(f"rank {r} loss {l_} vs {loss_ref}")
            q = r // P   # replica: its own microbatches' loss terms
            ce_ref = np.array([x for x, _ in per_ref[q * M:(q + 1) * M]])
            mse_ref = np.array([y for _, y in per_ref[q * M:(q + 1) * M]])
            if (np.linalg.norm(c_ - ce_ref) > tol * np.linalg.norm(ce_ref) or
                    np.linalg.norm(m_ - mse_ref) > tol * max(np.linalg.norm(mse_ref), 1e-30)):
                msgs.append(f"rank {r} per-microbatch loss terms differ")
            for n, v in g.items():
                ref = G_ref[n]
                e = np.linalg.norm(v - ref) / max(np.linalg.norm(ref), 1e-30)
                if e > tol:
                    msgs.append(f"rank {r} grad {n} rel err {e:.3e}")
        seen = set()
        for g, *_ in allg:
            seen |= set(g)
        missing = set(G_ref) - seen
        if missing:
            msgs.append(f"missing grads {sorted(missing)}")
        verdict = "PARITY OK" if not msgs else "PARITY FAIL"
        print(f"CASE {case} {verdict} loss {loss:.6f} oracle {loss_ref:.6f} sum_mode {rt.sum_mode} "
              f"{'; '.join(msgs[:8])}", flush=True)
    dist.barrier()
    rt.close()
    dist.barrier()


def hang_case(rank, world):
    """bm_step_wait: rank 1 skips its second step, so rank 0's second step blocks on a
    flag that never comes; rank 0 must get BM_E_TIMEOUT naming the blocked op."""
    from paper_2605_25451_b200 import _lib as L
    from paper_2605_25451_b200.runtime import Runtime
    cfg = get_config("C1", P=2, M=4, V=1)
    rt = Runtime(cfg, "f32", rank=rank, world=world)
    rt.load_weights(make_weights(cfg))
    db = rt.device_batch(make_batch(cfg))
    rt.step(db)
    rt.step_wait(60.0)
    dist.barrier()
    if rank == 1:
        time.sleep(25)      # keep the comm buffers mapped while rank 0 times out
        os._exit(0)
    rt.step(db)
    try:
        rt.step_wait(3.0)
        print("CASE hang NO TIMEOUT", flush=True)
    except L.BigMacError as e:
        ok = e.code == 10 and "blocked at op" in str(e)
        print(f"CASE hang {'TIMEOUT OK' if ok else 'TIMEOUT BAD'} {e}", flush=True)
    os._exit(0)   # the blocked device work dies with the context


def main():
    cases = sys.argv[1:]
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    # BM_TEST_ONE_GPU=1: every rank on cuda:0 (the single-GPU multi-rank fixture: CUDA
    # IPC works between processes of one device; the step-end sums then run over peer
    # memory, bm_ctx_init_peer_sum, because NCCL rejects duplicate devices)
    one_gpu = os.environ.get("BM_TEST_ONE_GPU") == "1"
    torch.cuda.set_device(0 if one_gpu else int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("gloo")
    if cases == ["hang"]:
        hang_case(rank, world)
    failed = False
    for case in cases:
        try:
            run_case(case, rank, world)
        except Exception:
            failed = True
            if rank == 0:
                print(f"CASE {case} PARITY ERROR {traceback.format_exc()[-1500:]!r}", flush=True)
            break   # the group's collective state is unknown after an exception
    dist.destroy_process_group()
    sys.exit(1 if failed else 0)


if __name__ == "__main__":
    main()
