"""Integer discrete-event simulation of a nested schedule (TEST INFRASTRUCTURE).

Semantics (SPEC S:297-301 read against P:362-364): each rank executes its
non-Send ops in program order on one compute resource; a compute op starts at
max(rank free, completion of its data producers); a Recv completes when its
matching Send has been issued; a Send is issued when its producer completes
(zero latency, unbounded slots).  Used by the oracle tests to check the
"no added bubble" claims under cost-weighted cuts.
"""
from __future__ import annotations

from .schedule import COMPUTE_KINDS, RECV, SEND, ScheduleError, E_DEADLOCK


def simulate(ranks, cost):
    """ranks: per-rank op lists (with comm ops); cost(rank, op) -> int >= 0.
    Returns (makespan, {(rank, index): (start, end)})."""
    P = len(ranks)
    ptr = [0] * P
    free = [0] * P
    sent = {}
    out = {}
    remaining = sum(len(x) for x in ranks)
    last_compute_end = [0] * P
    while remaining:
        progressed = False
        for r in range(P):
            ops = ranks[r]
            while ptr[r] < len(ops):
                i = ptr[r]
                op = ops[i]
                if op.kind == SEND:
                    t = last_compute_end[r]
                    sent[((r, op.peer, op.payload), op.seq)] = t
                    out[(r, i)] = (t, t)
                elif op.kind == RECV:
                    key = ((op.peer, r, op.payload), op.seq)
                    if key not in sent:
                        break
                    t = max(free[r], sent[key])
                    free[r] = t
                    out[(r, i)] = (t, t)
                else:
                    st = free[r]
                    en = st + cost(r, op)
                    free[r] = en
                    last_compute_end[r] = en
                    out[(r, i)] = (st, en)
                ptr[r] += 1
                remaining -= 1
                progressed = True
        if not progressed:
            raise ScheduleError(E_DEADLOCK, "simulation stalled")
    makespan = max(free) if free else 0
    return makespan, out


def uniform_cost(cf, cb, ef=0, eb=0, gf=0, gb=0):
    table = {"LlmFwd": cf, "LlmBwd": cb, "EncFwd": ef, "EncBwd": eb, "GenFwd": gf, "GenBwd": gb}

    def cost(r, op):
        return table[op.kind]
    return cost


def busy_time(ranks, cost, r):
    return sum(cost(r, op) for op in ranks[r] if op.kind in COMPUTE_KINDS)
