"""O-N: fp64 schedule interpreter over logical ranks (TEST INFRASTRUCTURE).

Executes the per-rank op lists that oracle.schedule.build emits, the way the
paper's executor does: an opcode stream per rank,
runtime buffers keyed by microbatch (+ virtual chunk), receive slots that a
Send fills and the consuming op releases, cross-module handoffs (encoder ->
entry stage gather, entry stage -> encoder scatter, last stage -> generator
scatter/gather) and gradient finalisation (sum of encoder/generator grads over
ranks) at schedule end.  All arithmetic is oracle.model's, so the
result must equal the sequential reference up to fp64 summation order.
Raises on buffer-miss, slot overwrite, stall and leaks.
"""
from __future__ import annotations

import numpy as np

from . import model as om
from .schedule import (ENC_FWD, ENC_BWD, LLM_FWD, LLM_BWD, GEN_FWD, GEN_BWD, SEND, RECV, LLM_W,
                       COMPUTE_KINDS, enc_owner, vstage)


class InterpError(Exception):
    pass


def run(sched, cfg, weights, batch):
    """cfg: synth ModelShape matching sched.cfg (P, M, V)."""
    sc = sched.cfg
    P, M, V = sc.stages, sc.microbatches, sc.vchunks
    assert (P, M, V) == (cfg.P, cfg.M, cfg.V)
    W = om.to_f64(weights)
    S = cfg.S
    gen_mode = sc.gen_place

    G = [dict() for _ in range(P)]
    enc_stash = [dict() for _ in range(P)]
    llm_stash = [dict() for _ in range(P)]
    gen_stash = [dict() for _ in range(P)]
    local = [dict() for _ in range(P)]          # same-rank handoffs
    slots = [dict() for _ in range(P)]          # (src, payload, slot) -> (seq, data)
    outbox = [dict() for _ in range(P)]         # peer -> list of (payload, seq, slot, data)
    pending_release = [dict() for _ in range(P)]  # op index -> list of slot keys
    ce = np.zeros(M)
    mse = np.zeros(M)
    ptr = [0] * P
    recv_data = [dict() for _ in range(P)]      # consumer-visible: (payload, mb) -> data list

    def shard(m, r):
        n = int(batch.n_gen[m])
        if gen_mode == "last_stage":
            return 0, n
        return om.shard_rows(n, P, r)

    def release_index(r, i, payload):
        ops = sched.ranks[r]
        j = i + 1
        while ops[j].kind not in COMPUTE_KINDS:
            j += 1
        if payload == "genin":
            while ops[j].kind != GEN_BWD:
                j += 1
        return j

    def take(r, payload, mb):
        key = (payload, mb)
        if key not in recv_data[r] or not recv_data[r][key]:
            raise InterpError(f"buffer miss: rank {r} {payload} mb {mb}")
        return recv_data[r][key]

    def exec_compute(r, i, op):
        m = op.mb
        if op.kind == ENC_FWD:
            E, cache = om.encoder_fwd(W, cfg, np.asarray(batch.patches[m], np.float64))
            enc_stash[r][m] = (cache, E)
            if r == 0:
                local[r][("emb", m)] = E
            return {"emb": E}
        if op.kind == ENC_BWD:
            if r == 0:
                dE = local[r].pop(("embgrad", m))
            else:
                dE = take(r, "embgrad", m)[0]
            cache, _ = enc_stash[r].pop(m)
            om.encoder_bwd(W, cfg, cache, dE, G[r])
            if r == 0:
                local[r].pop(("emb", m), None)
            return {}
        if op.kind == LLM_FWD:
            c = op.chunk
            s = vstage(P, r, c)
            if s == 0:
                n_mod = int(batch.n_mod[m])
                if sc.enc_place == "none":
                    raise InterpError("encoder placement 'none' unsupported by the interpreter")
                own = enc_owner(sc, m) == 0 if sc.enc_place == "dp_unit" else True
                emb = local[r][("emb", m)] if own else take(r, "emb", m)[0]
                x = om.embed_fwd(W, batch.ids[m], emb, n_mod)
            elif (s - 1) % P == r:
                x = local[r].pop(("act", m, s - 1))
            else:
                x = take(r, "act", m)[0]
            y, caches = om.llm_layers_fwd(W, cfg, om.stage_layers(cfg, s), np.array(x))
            ent = {"caches": caches}
            out = {}
            if s == P * V - 1:
                n_mod = int(batch.n_mod[m])
                Hn, ce_m, hcache = om.head_fwd(W, cfg, y, batch.labels[m], n_mod)
                ce[m] = ce_m
                ent["hcache"] = hcache
                ent["dHn"] = om.head_bwd_logits(W, cfg, hcache, 1.0 / M, G[r])
                n_gen = int(batch.n_gen[m])
                Xg = Hn[S - n_gen:]
                out["genin"] = {q: Xg[shard(m, q)[0]:shard(m, q)[1]].copy() for q in range(P)}
                local[r][("genin", m)] = out["genin"][r]
            else:
                if (s + 1) % P == r:
                    local[r][("act", m, s)] = y
                out["act"] = y
            llm_stash[r][(m, c)] = ent
            return out
        if op.kind == LLM_BWD:
            c = op.chunk
            s = vstage(P, r, c)
            zb = sc.llm_sched == "zb_h1"      # B = input gradient; stash kept until W (R23)
            ent = llm_stash[r][(m, c)] if zb else llm_stash[r].pop((m, c))
            if s == P * V - 1:
                dHn = ent["dHn"].copy()
                n_gen = int(batch.n_gen[m])
                base = S - n_gen
                if gen_mode == "dp_shard":
                    grads = {q: (local[r].pop(("gengrad", m)) if q == r else None) for q in range(P)}
                    others = take(r, "gengrad", m) if P > 1 else []
                    k = 0
                    for q in range(P):
                        if q != r:
                            grads[q] = others[k]
                            k += 1
                    for q in range(P):
                        lo, hi = shard(m, q)
                        dHn[base + lo:base + hi] += grads[q]
                elif gen_mode == "last_stage":
                    dHn[base:] += local[r].pop(("gengrad", m))
                dy = om.final_norm_bwd(W, ent["hcache"], dHn, G[r])
            elif (s + 1) % P == r:
                dy = local[r].pop(("grad", m, s + 1))
            else:
                dy = take(r, "grad", m)[0]
            if zb:
                ent["defer"] = []
            dx = om.llm_layers_bwd(W, cfg, om.stage_layers(cfg, s), ent["caches"], dy, G[r],
                                   ent.get("defer"))
            out = {}
            if s == 0:
                dE = om.embed_bwd(cfg, dx, batch.ids[m], int(batch.n_mod[m]), G[r])
                if sc.enc_place == "entry_stage" or enc_owner(sc, m) == 0:
                    local[r][("embgrad", m)] = dE
                out["embgrad"] = dE
            else:
                if (s - 1) % P == r:
                    local[r][("grad", m, s)] = dx
                out["grad"] = dx
            return out
        if op.kind == LLM_W:
            ent = llm_stash[r].pop((m, op.chunk))
            om.llm_wgrad(ent.pop("defer"), G[r])
            return {}
        if op.kind == GEN_FWD:
            lo, hi = shard(m, r)
            if r == P - 1:
                X = local[r].pop(("genin", m))
            else:
                X = take(r, "genin", m)[0]
            n_gen = int(batch.n_gen[m])
            t = np.asarray(batch.targets[m], np.float64)[lo:hi]
            part, cache = om.gen_fwd(W, cfg, X, t, float(n_gen * cfg.d_t))
            mse[m] += part
            gen_stash[r][m] = cache
            return {}
        if op.kind == GEN_BWD:
            cache = gen_stash[r].pop(m)
            dX = om.gen_bwd(W, cfg, cache, 1.0 / M, G[r])
            if r == P - 1:
                local[r][("gengrad", m)] = dX
            return {"gengrad": dX}
        raise InterpError(op.kind)

    last_out = [dict() for _ in range(P)]
    total = sum(len(x) for x in sched.ranks)
    done = 0
    while done < total:
        progressed = False
        for r in range(P):
            ops = sched.ranks[r]
            while ptr[r] < len(ops):
                i = ptr[r]
                op = ops[i]
                if op.kind == SEND:
                    data = last_out[r][op.payload]
                    if op.payload == "genin":
                        data = data[op.peer]
                    outbox[r].setdefault(op.peer, []).append((op.payload, op.seq, op.slot, np.array(data), op.mb))
                elif op.kind == RECV:
                    key = (op.peer, op.payload, op.slot)
                    if key not in slots[r] or slots[r][key][0] != op.seq:
                        break
                    data = slots[r][key][1]
                    recv_data[r].setdefault((op.payload, op.mb), []).append(data)
                    j = release_index(r, i, op.payload)
                    pending_release[r].setdefault(j, []).append((key, op.payload, op.mb))
                else:
                    last_out[r] = exec_compute(r, i, op)
                    for key, payload, mb in pending_release[r].pop(i, []):
                        del slots[r][key]
                        lst = recv_data[r][(payload, mb)]
                        lst.pop(0)
                        if not lst:
                            del recv_data[r][(payload, mb)]
                ptr[r] += 1
                done += 1
                progressed = True
            # drain outboxes (per-peer FIFO; blocked while the slot is occupied)
        for r in range(P):
            for peer, q in outbox[r].items():
                while q:
                    payload, seq, slot, data, mb = q[0]
                    key = (r, payload, slot)
                    if key in slots[peer]:
                        break
                    slots[peer][key] = (seq, data)
                    q.pop(0)
                    progressed = True
        if not progressed:
            raise InterpError("interpreter stalled (deadlock)")
    # drain remaining messages
    for r in range(P):
        for peer, q in outbox[r].items():
            if q:
                raise InterpError("undelivered messages at end")
    for r in range(P):
        if slots[r] or enc_stash[r] or llm_stash[r] or gen_stash[r] or local[r] or recv_data[r]:
            raise InterpError(f"leak on rank {r}: slots={list(slots[r])} local={list(local[r])}")

    # finalize: sum encoder/generator grads over ranks
    grads = {}
    for r in range(P):
        for k, v in G[r].items():
            grads[k] = grads[k] + v if k in grads else v.copy()
    for k in W:
        if k not in grads:
            grads[k] = np.zeros_like(W[k])
    per_mb = list(zip(ce.tolist(), mse.tolist()))
    loss = float(np.sum(ce + mse) / M)
    return loss, per_mb, grads, G
