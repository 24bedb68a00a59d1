"""Exhaustive searches on tiny configurations (TEST INFRASTRUCTURE).

1. min_peak_encoder_window: over ALL interleavings of EncFwd(u)/EncBwd(u)
   into the rank-0 LLM list that are dependency-safe (EncFwd(u) before F_u,
   EncBwd(u) after G_u, FIFO per kind) the minimum possible peak number of live
   encoder units.  BigMac with W = W* must attain it.
2. free_placement_makespan: over ALL per-rank placements of encoder units
   (not restricted to full-width cuts) the minimum DES makespan; documents
   SURVEY §8(c) Q14 (BigMac is optimal within the cut class, not globally).
"""
from __future__ import annotations

import itertools

from .schedule import llm_base_schedule, Op, LLM_FWD, LLM_BWD, ENC_FWD, ENC_BWD, SEND, RECV
from .schedule import SchedCfg, verify_dependencies
from .des import simulate


def min_peak_encoder_window(P: int, M: int, V: int) -> int:
    base0 = llm_base_schedule(P, M, V)[0]
    n_u = M // P
    F = {u: base0.index(("F", u * P, 0)) for u in range(n_u)}
    G = {u: base0.index(("B", u * P + P - 1, 0)) for u in range(n_u)}
    L = len(base0)
    best = [10 ** 9]

    def rec(i, nf, nb, live, peak):
        # i: LLM ops emitted; nf/nb: EncFwd/EncBwd emitted
        if peak >= best[0]:
            return
        if i == L and nf == n_u and nb == n_u:
            best[0] = peak
            return
        # emit next LLM op if its encoder input is ready
        if i < L:
            ok = True
            for u in range(n_u):
                if F[u] == i and nf <= u:
                    ok = False
            if ok:
                rec(i + 1, nf, nb, live, peak)
        # emit EncFwd(nf)
        if nf < n_u:
            rec(i, nf + 1, nb, live + 1, max(peak, live + 1))
        # emit EncBwd(nb) if its gradient exists (G_nb emitted) and fwd done
        if nb < nf and G[nb] < i:
            rec(i, nf, nb + 1, live - 1, peak)

    rec(0, 0, 0, 0, 0)
    return best[0]


def free_placement_makespan(P: int, M: int, ef: int, eb: int, cf: int = 1, cb: int = 1,
                            limit: int = 200000):
    """Minimum makespan over every per-rank insertion of EncFwd(u)/EncBwd(u)
    (V = 1, no generator, zero-latency comm), keeping each rank's LLM order."""
    base = llm_base_schedule(P, M, 1)
    n_u = M // P
    cfg = SchedCfg(P, M, 1, warmup_units=n_u, gen_place="none")

    def placements(r):
        L = len(base[r])
        # choose positions (in the merged list) for n_u fwd and n_u bwd ops
        llm = [Op(LLM_FWD if k == "F" else LLM_BWD, mb=m, chunk=c) for k, m, c in base[r]]
        total = L + 2 * n_u
        for slots in itertools.combinations(range(total), 2 * n_u):
            for order in _enc_orders(n_u):
                merged, it_l, it_e = [], iter(llm), iter(order)
                sset = set(slots)
                for p in range(total):
                    merged.append(next(it_e) if p in sset else next(it_l))
                yield [(o if o.kind not in (ENC_FWD, ENC_BWD) else Op(o.kind, mb=o.unit * P + r, unit=o.unit))
                       for o in merged]

    best = None
    count = 0
    per_rank = [list(placements(r)) for r in range(P)]
    for combo in itertools.product(*per_rank):
        count += 1
        if count > limit:
            break
        lists = [list(x) for x in combo]
        if verify_dependencies(cfg, lists):
            continue
        ranks = _with_comm_free(cfg, lists)
        mk, _ = simulate(ranks, lambda r, op: {"LlmFwd": cf, "LlmBwd": cb, "EncFwd": ef, "EncBwd": eb}[op.kind])
        best = mk if best is None else min(best, mk)
    return best


def _enc_orders(n_u):
    """All valid sequences of EncFwd(0..)/EncBwd(0..) with FIFO per kind and
    EncBwd(u) after EncFwd(u)."""
    out = []

    def rec(nf, nb, acc):
        if nf == n_u and nb == n_u:
            out.append(list(acc))
            return
        if nf < n_u:
            acc.append(Op(ENC_FWD, unit=nf))
            rec(nf + 1, nb, acc)
            acc.pop()
        if nb < nf:
            acc.append(Op(ENC_BWD, unit=nb))
            rec(nf, nb + 1, acc)
            acc.pop()
    rec(0, 0, [])
    return out


def _with_comm_free(cfg, lists):
    from .schedule import insert_comm
    ranks, _ = insert_comm(cfg, lists)
    return ranks
