"""O-S: the schedule oracle (TEST INFRASTRUCTURE; see oracle/__init__.py).

Plain, slow, step-by-step implementation of BigMac's scheduler:
  get_llm_schedule      P:309-310, P:133 (1F1B), P:200 (interleaved 1F1B)
  cut timeline          P:199, P:257 ("columns"; reading SURVEY §8(c) Q1)
  build_schedule        P:247-271 (Fig. build_schedule)
  insert_comm_ops
  deadlock_check        P:317 (+ credit-ring sizing)
  order property
  zero-bubble base      P:552-556 names zero-bubble pipeline parallelism (Qi et al.)
                        as the next LLM schedule class; ZB-H1 built as in DESIGN.md R23
  decoupled CP          P:388-398: distinct LLM / encoder CP degrees, encoder unit of
                        P llm_cp / enc_cp microbatches, CP-conversion all-to-all
                        (build_cp; schedule level, R25)
Every reading of an ambiguous passage is listed in DESIGN.md "Readings".
"""
from __future__ import annotations

from collections import deque
from dataclasses import dataclass, field

# status codes mirror include/bigmac.h bm_status
OK, E_INVALID, E_REMAINDER, E_WARMUP, E_DEPENDENCY, E_DEADLOCK = 0, 1, 2, 3, 4, 5


class ScheduleError(Exception):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


# op kinds and payloads (names are the serialization tokens)
ENC_FWD, ENC_BWD, LLM_FWD, LLM_BWD, GEN_FWD, GEN_BWD, SEND, RECV, LLM_W = (
    "EncFwd", "EncBwd", "LlmFwd", "LlmBwd", "GenFwd", "GenBwd", "Send", "Recv", "LlmW")
# LLM_W: the weight-gradient half of an LLM backward (zero-bubble schedules, R23);
# under zb_h1 LLM_BWD computes only the input gradient
COMPUTE_KINDS = (ENC_FWD, ENC_BWD, LLM_FWD, LLM_BWD, GEN_FWD, GEN_BWD, LLM_W)
LLM_KIND = {"F": LLM_FWD, "B": LLM_BWD, "W": LLM_W}
PAYLOADS = ("act", "grad", "emb", "embgrad", "genin", "gengrad")


@dataclass(frozen=True)
class Op:
    kind: str
    mb: int = -1
    chunk: int = -1
    unit: int = -1
    peer: int = -1
    payload: str = ""
    slot: int = -1
    seq: int = -1


@dataclass
class SchedCfg:
    stages: int                 # P  (pp_size)
    microbatches: int           # M  (microbatch_num)
    vchunks: int = 1            # V  (vpp size)
    warmup_units: int = 0       # W; 0 => W*
    llm_sched: str = "1f1b"     # "1f1b" | "interleaved" | "zb_h1" (R23)
    enc_place: str = "dp_unit"  # "none" | "dp_unit" | "entry_stage"
    gen_place: str = "dp_shard" # "none" | "dp_shard" | "last_stage"
    cost_fwd: int = 1           # cut-timeline cost ratio, default 1:2
    cost_bwd: int = 2
    ring_slack: int = 1         # extra receive slots per channel above the minimum
    enc_exclude: int = 0        # bit mask of ranks running no encoder microbatches (DESIGN R22)
    cost_wgrad: int = 0         # zb_h1: W's share of cost_bwd; 0 => cost_bwd // 2 (R23)
    llm_cp: int = 1             # LLM context-parallel degree (R25)
    enc_cp: int = 1             # encoder context-parallel degree


@dataclass
class Stats:
    w_star: int
    warmup_units: int
    peak_enc_units: int
    peak_gen_shards: int
    peak_llm_inflight: int
    llm_idle_cost_units: int
    makespan_cost_units: int
    n_ops: int
    ring_slots: dict


@dataclass
class Schedule:
    cfg: SchedCfg
    ranks: list                 # P lists of Op (compute + comm)
    stats: list                 # P Stats
    rings: dict = field(default_factory=dict)   # (src, dst, payload) -> K
    llm_base: list = field(default_factory=list)
    times: dict = field(default_factory=dict)   # (rank, kind, mb, chunk) -> (start, end)


# ----------------------------------------------------------------------------
# 1. validation
# ----------------------------------------------------------------------------
def validate(cfg: SchedCfg) -> None:
    P, M, V = cfg.stages, cfg.microbatches, cfg.vchunks
    if P < 1 or M < 1 or V < 1 or cfg.warmup_units < 0:
        raise ScheduleError(E_INVALID, "P, M, V must be >= 1 and W >= 0")
    if cfg.cost_fwd < 1 or cfg.cost_bwd < 1 or cfg.ring_slack < 0:
        raise ScheduleError(E_INVALID, "costs must be >= 1 and ring_slack >= 0")
    if cfg.llm_sched == "1f1b" and V != 1:
        raise ScheduleError(E_INVALID, "1F1B requires V == 1")
    if cfg.llm_sched == "interleaved" and V < 2:
        raise ScheduleError(E_INVALID, "interleaved 1F1B requires V >= 2")
    if cfg.llm_sched not in ("1f1b", "interleaved", "zb_h1"):
        raise ScheduleError(E_INVALID, "unknown llm_sched")
    if cfg.cost_wgrad < 0:
        raise ScheduleError(E_INVALID, "cost_wgrad must be >= 0")
    if cfg.llm_sched == "zb_h1":
        if V != 1:
            raise ScheduleError(E_INVALID, "ZB-H1 requires V == 1")
        if not 1 <= wgrad_cost(cfg) < cfg.cost_bwd:
            raise ScheduleError(E_INVALID, "ZB-H1 needs 1 <= W cost < cost_bwd (B and W both >= 1)")
    if cfg.enc_place not in ("none", "dp_unit", "entry_stage"):
        raise ScheduleError(E_INVALID, "unknown enc_place")
    if cfg.gen_place not in ("none", "dp_shard", "last_stage"):
        raise ScheduleError(E_INVALID, "unknown gen_place")
    if cfg.llm_cp < 1 or cfg.enc_cp < 1 or cfg.enc_cp > cfg.llm_cp or (P * cfg.llm_cp) % cfg.enc_cp:
        # the unit is enlarged from P to P llm_cp / enc_cp microbatches: enc_cp <= llm_cp
        raise ScheduleError(E_INVALID, "need 1 <= enc_cp <= llm_cp and enc_cp dividing P * llm_cp")
    cp = cfg.llm_cp > 1 or cfg.enc_cp > 1
    if cp and (cfg.enc_place == "entry_stage" or cfg.gen_place == "dp_shard" or cfg.enc_exclude):
        raise ScheduleError(E_INVALID, "decoupled CP: enc_place none / dp_unit, gen_place none / last_stage, "
                                       "no enc_exclude")
    unit = P * cfg.llm_cp // cfg.enc_cp
    if M % unit != 0:
        # units of pp_size (x llm_cp / enc_cp) micro-batches
        raise ScheduleError(E_REMAINDER, f"M={M} is not a multiple of the encoder unit {unit}")
    if cfg.enc_exclude:
        full = (1 << P) - 1
        if cfg.enc_exclude < 0 or cfg.enc_exclude & ~full or cfg.enc_exclude == full:
            raise ScheduleError(E_INVALID, "enc_exclude: a mask of ranks < P leaving at least one rank")
        if cfg.enc_place != "dp_unit":
            raise ScheduleError(E_INVALID, "enc_exclude applies to the DP encoder units")


def wgrad_cost(cfg: SchedCfg) -> int:
    """Cost of the W half of a backward under zb_h1 (the B half costs cost_bwd - W)."""
    return cfg.cost_wgrad if cfg.cost_wgrad > 0 else cfg.cost_bwd // 2


def enc_owner(cfg: SchedCfg, m: int) -> int:
    """Rank that runs microbatch m's encoder (reading R3: mb uP+r on rank r);
    a rank in enc_exclude hands its microbatch to the nearest lower rank not in the
    mask, cyclically (reading R22)."""
    P = cfg.stages
    r = m % P
    while (cfg.enc_exclude >> r) & 1:
        r = (r - 1) % P
    return r


# ----------------------------------------------------------------------------
# 2. LLM base schedule (get_llm_schedule)
# ----------------------------------------------------------------------------
def llm_base_schedule(P: int, M: int, V: int):
    """Per-rank lists of ('F'|'B', mb, chunk) — Megatron-style 1F1B / interleaved."""
    out = []
    for r in range(P):
        if V == 1:
            w = min(P - r - 1, M)
            fwd = [(m, 0) for m in range(M)]
            bwd = [(m, 0) for m in range(M)]
        else:
            w = min(2 * (P - r - 1) + (V - 1) * P, M * V)
            fwd, bwd = [], []
            for k in range(M * V):
                g, j = divmod(k, P * V)
                c = j // P
                m = g * P + (j % P)
                fwd.append((m, c))
                bwd.append((m, V - 1 - c))
        total = len(fwd)
        ops = [("F",) + fwd[k] for k in range(w)]
        for i in range(total - w):
            ops.append(("F",) + fwd[w + i])
            ops.append(("B",) + bwd[i])
        for i in range(total - w, total):
            ops.append(("B",) + bwd[i])
        out.append(ops)
    return out


def zb_h1_schedule(P: int, M: int, cf: int, cb: int, cw: int):
    """Per-rank lists of ('F'|'B'|'W', mb, 0) for the ZB-H1 zero-bubble schedule
    (R23; P:552-556 points to Qi et al.'s zero-bubble pipelines).
    The backward is split into B (input gradient, cost cb) and W (weight
    gradient, cost cw).  Every rank keeps the 1F1B order of its F and B ops
    (warmup min(P-r-1, M)) and holds at most P microbatches between F and W (the
    1F1B peak of rank 0, so no rank needs more activation memory than 1F1B's
    busiest one).  Built by simulating the ranks in time order; a rank free at
    time t does, in this order of preference:
      1. its next F if P microbatches are held -> the oldest pending W instead;
      2. its next F/B if its producer has finished by t;
      3. the oldest pending W if it ends no later than the earliest time the
         next F/B can start (the producer's end if it is scheduled, else the
         producer rank's free time plus the producer's cost), so a W fills
         idle time without delaying the F/B chain;
      4. nothing until t + 1.
    After its last B it runs the pending W's oldest first."""
    fb = []
    for r in range(P):
        w = min(P - r - 1, M)
        ops = [("F", m) for m in range(w)]
        for i in range(M - w):
            ops += [("F", w + i), ("B", i)]
        ops += [("B", i) for i in range(M - w, M)]
        fb.append(ops)
    end = {}
    lists = [[] for _ in range(P)]
    t = [0] * P
    ptr = [0] * P
    pending = [deque() for _ in range(P)]
    held = [0] * P
    active = set(range(P))

    def run_w(r):
        m = pending[r].popleft()
        lists[r].append(("W", m, 0))
        end[(r, "W", m)] = t[r] + cw
        t[r] += cw
        held[r] -= 1

    while active:
        r = min(active, key=lambda x: (t[x], x))   # every other rank is free at >= t[r]
        if ptr[r] == len(fb[r]):
            if pending[r]:
                run_w(r)
            else:
                active.discard(r)
            continue
        k, m = fb[r][ptr[r]]
        if k == "F" and held[r] >= P:
            run_w(r)
            continue
        dep = None
        if k == "F" and r > 0:
            dep, dep_cost = (r - 1, "F", m), cf
        if k == "B" and r < P - 1:
            dep, dep_cost = (r + 1, "B", m), cb
        if dep is None or (dep in end and end[dep] <= t[r]):
            lists[r].append((k, m, 0))
            end[(r, k, m)] = t[r] + (cf if k == "F" else cb)
            t[r] = end[(r, k, m)]
            ptr[r] += 1
            if k == "F":
                held[r] += 1
            else:
                pending[r].append(m)
        else:
            q = dep[0]
            earliest = end[dep] if dep in end else max(t[r], t[q]) + dep_cost
            if pending[r] and t[r] + cw <= earliest:
                run_w(r)
            else:
                t[r] += 1
    return lists


def vstage(P: int, rank: int, chunk: int) -> int:
    return chunk * P + rank


# ----------------------------------------------------------------------------
# 3. cut timeline: integer DES of the LLM lists
# ----------------------------------------------------------------------------
def des_llm(base, P: int, V: int, cf: int, cb: int, cw: int = 0):
    """start/end of every LLM op with per-rank program order and data deps
    F(m,s) <- F(m,s-1),  B(m,s) <- B(m,s+1) (and F(m,s) by program order;
    W(m,s), zb_h1 only, follows B(m,s) by program order and costs cw).
    Returns {(r, 'F'|'B'|'W', m, c): (start, end)}; raises E_DEPENDENCY on stall."""
    times = {}
    ptr = [0] * P
    free = [0] * P
    remaining = sum(len(l) for l in base)
    while remaining:
        progressed = False
        for r in range(P):
            while ptr[r] < len(base[r]):
                k, m, c = base[r][ptr[r]]
                s = vstage(P, r, c)
                dep = None
                if k == "F" and s > 0:
                    dep = ((s - 1) % P, "F", m, (s - 1) // P)
                if k == "B" and s < P * V - 1:
                    dep = ((s + 1) % P, "B", m, (s + 1) // P)
                if dep is not None and dep not in times:
                    break
                st = max(free[r], times[dep][1] if dep is not None else 0)
                en = st + {"F": cf, "B": cb, "W": cw}[k]
                times[(r, k, m, c)] = (st, en)
                free[r] = en
                ptr[r] += 1
                remaining -= 1
                progressed = True
        if not progressed:
            raise ScheduleError(E_DEPENDENCY, "LLM base schedule stalls")
    return times


# ----------------------------------------------------------------------------
# 4-5. nesting (build_schedule)
# ----------------------------------------------------------------------------
def w_star(base0, P: int) -> int:
    """Minimal warmup: max_i |{j >= i : F_j precedes G_i in the rank-0 list}|
    with F_i = F(iP, chunk 0)@0 and G_i = B(iP+P-1, chunk 0)@0."""
    pos = {(k, m, c): i for i, (k, m, c) in enumerate(base0)}
    M = max(m for _, m, _ in base0) + 1
    n_u = M // P
    best = 1
    for i in range(n_u):
        g = pos[("B", i * P + P - 1, 0)]
        cnt = sum(1 for j in range(i, n_u) if pos[("F", j * P, 0)] < g)
        best = max(best, cnt)
    return best


def nest(cfg: SchedCfg, base, times):
    """Compute-op lists per rank (O-S steps 4-5)."""
    P, M, V = cfg.stages, cfg.microbatches, cfg.vchunks
    n_u = M // P
    entry = cfg.enc_place == "entry_stage"
    W = 0 if entry else (cfg.warmup_units if cfg.warmup_units > 0 else w_star(base[0], P))
    enc = cfg.enc_place == "dp_unit"
    gen = cfg.gen_place

    events = []
    for r in range(P):
        for (k, m, c) in base[r]:
            st, _ = times[(r, k, m, c)]
            events.append((st, 2, r, (r, k, m, c)))
    if gen != "none":
        for m in range(M):
            _, en = times[(P - 1, "F", m, V - 1)]
            events.append((en, 0, m, ("GEN", m)))
    if enc:
        for u in range(n_u):
            _, en = times[(0, "B", u * P + P - 1, 0)]
            events.append((en, 1, u, ("ENC", u)))
    events.sort(key=lambda e: (e[0], e[1], e[2]))

    lists = [[] for _ in range(P)]
    nxt = 0

    def unit_ops(kind, u):   # the unit's encoder microbatches on every rank, each rank in mb order
        for r in range(P):
            for m in range(u * P, u * P + P):
                if enc_owner(cfg, m) == r:
                    lists[r].append(Op(kind, mb=m, unit=u))
    if enc:
        for u in range(min(W, n_u)):
            unit_ops(ENC_FWD, u)
        nxt = min(W, n_u)
    for _, cls, _, ev in events:
        if cls == 2:
            r, k, m, c = ev
            if enc and k == "F" and r == 0 and c == 0 and m // P >= nxt:
                raise ScheduleError(
                    E_WARMUP, f"W={W} too small: F({m},0)@0 precedes EncFwd({m // P})")
            # memory-efficient baseline (Fig. 3): the encoder is the entry
            # stage's first layers -- EncFwd(m) right before F(m,0), EncBwd(m) right after B(m,0)
            if entry and k == "F" and r == 0 and c == 0:
                lists[r].append(Op(ENC_FWD, mb=m, unit=m))
            lists[r].append(Op(LLM_KIND[k], mb=m, chunk=c))
            if entry and k == "B" and r == 0 and c == 0:
                lists[r].append(Op(ENC_BWD, mb=m, unit=m))
        elif cls == 0:
            m = ev[1]
            targets = range(P) if gen == "dp_shard" else [P - 1]
            for r in targets:
                lists[r].append(Op(GEN_FWD, mb=m))
                lists[r].append(Op(GEN_BWD, mb=m))
        else:
            u = ev[1]
            unit_ops(ENC_BWD, u)
            if nxt < n_u:
                unit_ops(ENC_FWD, nxt)
                nxt += 1
    return lists, W


# ----------------------------------------------------------------------------
# 6. communication operators (insert_comm_ops)
# ----------------------------------------------------------------------------
def _recvs_before(cfg: SchedCfg, r: int, op: Op):
    P, V = cfg.stages, cfg.vchunks
    out = []
    if op.kind == LLM_FWD:
        s = vstage(P, r, op.chunk)
        if s > 0 and (s - 1) % P != r:
            out.append(Op(RECV, mb=op.mb, chunk=op.chunk, peer=(s - 1) % P, payload="act"))
        if s == 0 and cfg.enc_place == "dp_unit" and enc_owner(cfg, op.mb) != 0:
            out.append(Op(RECV, mb=op.mb, unit=op.mb // P, peer=enc_owner(cfg, op.mb), payload="emb"))
    elif op.kind == LLM_BWD:
        s = vstage(P, r, op.chunk)
        if s < P * V - 1 and (s + 1) % P != r:
            out.append(Op(RECV, mb=op.mb, chunk=op.chunk, peer=(s + 1) % P, payload="grad"))
        if s == P * V - 1 and cfg.gen_place == "dp_shard":
            for q in range(P):
                if q != r:
                    out.append(Op(RECV, mb=op.mb, peer=q, payload="gengrad"))
    elif op.kind == ENC_BWD and r != 0 and cfg.enc_place == "dp_unit":
        out.append(Op(RECV, mb=op.mb, unit=op.unit, peer=0, payload="embgrad"))
    elif op.kind == GEN_FWD and cfg.gen_place == "dp_shard" and r != P - 1:
        out.append(Op(RECV, mb=op.mb, peer=P - 1, payload="genin"))
    return out


def _sends_after(cfg: SchedCfg, r: int, op: Op):
    P, V = cfg.stages, cfg.vchunks
    out = []
    if op.kind == LLM_FWD:
        s = vstage(P, r, op.chunk)
        if s < P * V - 1 and (s + 1) % P != r:
            out.append(Op(SEND, mb=op.mb, chunk=op.chunk, peer=(s + 1) % P, payload="act"))
        if s == P * V - 1 and cfg.gen_place == "dp_shard":
            for q in range(P):
                if q != r:
                    out.append(Op(SEND, mb=op.mb, peer=q, payload="genin"))
    elif op.kind == LLM_BWD:
        s = vstage(P, r, op.chunk)
        if s > 0 and (s - 1) % P != r:
            out.append(Op(SEND, mb=op.mb, chunk=op.chunk, peer=(s - 1) % P, payload="grad"))
        if s == 0 and cfg.enc_place == "dp_unit" and enc_owner(cfg, op.mb) != 0:
            out.append(Op(SEND, mb=op.mb, unit=op.mb // P, peer=enc_owner(cfg, op.mb), payload="embgrad"))
    elif op.kind == ENC_FWD and r != 0 and cfg.enc_place == "dp_unit":
        out.append(Op(SEND, mb=op.mb, unit=op.unit, peer=0, payload="emb"))
    elif op.kind == GEN_BWD and cfg.gen_place == "dp_shard" and r != P - 1:
        out.append(Op(SEND, mb=op.mb, peer=P - 1, payload="gengrad"))
    return out


def insert_comm(cfg: SchedCfg, lists):
    """Recv immediately before its consumer, Send immediately after its producer;
    per-channel sequence numbers in program order (channel = (src, dst, payload))."""
    P = cfg.stages
    out = []
    for r in range(P):
        ops = []
        for op in lists[r]:
            ops.extend(_recvs_before(cfg, r, op))
            ops.append(op)
            ops.extend(_sends_after(cfg, r, op))
        out.append(ops)
    # sequence numbers
    send_cnt, recv_cnt = {}, {}
    for r in range(P):
        for i, op in enumerate(out[r]):
            if op.kind == SEND:
                ch = (r, op.peer, op.payload)
                j = send_cnt.get(ch, 0)
                send_cnt[ch] = j + 1
                out[r][i] = _with(op, seq=j)
            elif op.kind == RECV:
                ch = (op.peer, r, op.payload)
                j = recv_cnt.get(ch, 0)
                recv_cnt[ch] = j + 1
                out[r][i] = _with(op, seq=j)
    if send_cnt != recv_cnt:
        raise ScheduleError(E_DEPENDENCY, "unmatched send/recv counts")
    return out, send_cnt


def _with(op: Op, **kw) -> Op:
    d = dict(kind=op.kind, mb=op.mb, chunk=op.chunk, unit=op.unit, peer=op.peer,
             payload=op.payload, slot=op.slot, seq=op.seq)
    d.update(kw)
    return Op(**d)


# ----------------------------------------------------------------------------
# 6b. happens-before graph, credit rings and deadlock check
# ----------------------------------------------------------------------------
def _index(lists):
    """Node ids, message locations and release ops."""
    P = len(lists)
    nid = {}
    n = 0
    for r in range(P):
        for i in range(len(lists[r])):
            nid[(r, i)] = n
            n += 1
    send_at, recv_at, release_at = {}, {}, {}
    for r in range(P):
        ops = lists[r]
        for i, op in enumerate(ops):
            if op.kind == SEND:
                send_at[((r, op.peer, op.payload), op.seq)] = (r, i)
            elif op.kind == RECV:
                ch = (op.peer, r, op.payload)
                recv_at[(ch, op.seq)] = (r, i)
                # consumer = first compute op after the Recv
                j = i + 1
                while ops[j].kind not in COMPUTE_KINDS:
                    j += 1
                if op.payload == "genin":
                    # the generator input is read by GenFwd and GenBwd
                    while ops[j].kind != GEN_BWD:
                        j += 1
                release_at[(ch, op.seq)] = (r, j)
    return nid, n, send_at, recv_at, release_at


def _base_edges(lists, nid, send_at, recv_at):
    """(a) non-Send chain per rank, (b) Send chain per (rank, peer),
    (c) producer -> Send, (d) Send -> Recv."""
    edges = []
    for r, ops in enumerate(lists):
        prev = None
        last_send = {}
        for i, op in enumerate(ops):
            if op.kind == SEND:
                if prev is not None:
                    edges.append((nid[(r, prev)], nid[(r, i)]))
                if op.peer in last_send:
                    edges.append((nid[(r, last_send[op.peer])], nid[(r, i)]))
                last_send[op.peer] = i
            else:
                if prev is not None:
                    edges.append((nid[(r, prev)], nid[(r, i)]))
                prev = i
    for key, (r, i) in send_at.items():
        rr, ri = recv_at[key]
        edges.append((nid[(r, i)], nid[(rr, ri)]))
    return edges


def _credit_edges(ch, K, nmsg, nid, send_at, release_at):
    out = []
    for j in range(K, nmsg):
        a = release_at[(ch, j - K)]
        b = send_at[(ch, j)]
        out.append((nid[a], nid[b]))
    return out


def _acyclic(n, edges) -> bool:
    adj = [[] for _ in range(n)]
    indeg = [0] * n
    for a, b in edges:
        adj[a].append(b)
        indeg[b] += 1
    q = deque(i for i in range(n) if indeg[i] == 0)
    seen = 0
    while q:
        x = q.popleft()
        seen += 1
        for y in adj[x]:
            indeg[y] -= 1
            if indeg[y] == 0:
                q.append(y)
    return seen == n


def size_rings(cfg: SchedCfg, lists, counts):
    """Per channel: the smallest K such that program order + data + this
    channel's credit edges (release(j-K) -> send(j)) stay acyclic, plus
    `ring_slack`, capped at the message count; then bump all channels until
    the combined graph is acyclic (deadlock-free under eager push)."""
    nid, n, send_at, recv_at, release_at = _index(lists)
    base = _base_edges(lists, nid, send_at, recv_at)
    if not _acyclic(n, base):
        raise ScheduleError(E_DEADLOCK, "schedule deadlocks even with unbounded slots")
    rings = {}
    for ch in sorted(counts):
        nmsg = counts[ch]
        K = 1
        while K < nmsg and not _acyclic(n, base + _credit_edges(ch, K, nmsg, nid, send_at, release_at)):
            K += 1
        rings[ch] = min(K + cfg.ring_slack, nmsg)
    while True:
        allc = []
        for ch in sorted(counts):
            allc += _credit_edges(ch, rings[ch], counts[ch], nid, send_at, release_at)
        if _acyclic(n, base + allc):
            break
        grew = False
        for ch in sorted(counts):
            if rings[ch] < counts[ch]:
                rings[ch] += 1
                grew = True
        if not grew:  # pragma: no cover - unreachable (base graph is acyclic)
            raise ScheduleError(E_DEADLOCK, "credit rings cannot be sized")
    return rings


def assign_slots(lists, rings):
    out = []
    for r, ops in enumerate(lists):
        new = []
        for op in ops:
            if op.kind == SEND:
                op = _with(op, slot=op.seq % rings[(r, op.peer, op.payload)])
            elif op.kind == RECV:
                op = _with(op, slot=op.seq % rings[(op.peer, r, op.payload)])
            new.append(op)
        out.append(new)
    return out


# ----------------------------------------------------------------------------
# 7. verification and statistics
# ----------------------------------------------------------------------------
def compute_deps(cfg: SchedCfg, r: int, op: Op):
    """Data producers of a compute op as (rank, kind, mb, chunk-or-unit) keys."""
    P, V = cfg.stages, cfg.vchunks
    deps = []
    if op.kind == LLM_FWD:
        s = vstage(P, r, op.chunk)
        if s > 0:
            deps.append(((s - 1) % P, LLM_FWD, op.mb, (s - 1) // P))
        elif cfg.enc_place == "dp_unit":
            deps.append((enc_owner(cfg, op.mb), ENC_FWD, op.mb, -1))
        elif cfg.enc_place == "entry_stage":
            deps.append((0, ENC_FWD, op.mb, -1))
    elif op.kind == LLM_BWD:
        s = vstage(P, r, op.chunk)
        deps.append((r, LLM_FWD, op.mb, op.chunk))
        if s < P * V - 1:
            deps.append(((s + 1) % P, LLM_BWD, op.mb, (s + 1) // P))
        elif cfg.gen_place == "dp_shard":
            deps += [(q, GEN_BWD, op.mb, -1) for q in range(P)]
        elif cfg.gen_place == "last_stage":
            deps.append((P - 1, GEN_BWD, op.mb, -1))
    elif op.kind == LLM_W:
        deps.append((r, LLM_BWD, op.mb, op.chunk))
    elif op.kind == ENC_BWD:
        deps.append((r, ENC_FWD, op.mb, -1))
        deps.append((0, LLM_BWD, op.mb, 0))
    elif op.kind == GEN_FWD:
        deps.append((P - 1, LLM_FWD, op.mb, V - 1))
    elif op.kind == GEN_BWD:
        deps.append((r, GEN_FWD, op.mb, -1))
    return deps


def _ckey(r, op):
    return (r, op.kind, op.mb, op.chunk if op.kind in (LLM_FWD, LLM_BWD, LLM_W) else -1)


def verify_dependencies(cfg: SchedCfg, lists):
    """Empty list iff a global order exists in which every compute op's data
    producers complete first; otherwise the data edges of one cycle (or the
    missing producers)."""
    P = cfg.stages
    comp = [[op for op in ops if op.kind in COMPUTE_KINDS] for ops in lists]
    nid, n = {}, 0
    for r in range(P):
        for op in comp[r]:
            k = _ckey(r, op)
            if k in nid:
                return [("duplicate", k)]
            nid[k] = n
            n += 1
    edges, data = [], {}
    for r in range(P):
        for i, op in enumerate(comp[r]):
            if i:
                edges.append((nid[_ckey(r, comp[r][i - 1])], nid[_ckey(r, op)]))
            for d in compute_deps(cfg, r, op):
                if d not in nid:
                    return [("missing", d, _ckey(r, op))]
                e = (nid[d], nid[_ckey(r, op)])
                edges.append(e)
                data[e] = (d, _ckey(r, op))
    # find a cycle (iterative DFS)
    adj = [[] for _ in range(n)]
    for a, b in edges:
        adj[a].append(b)
    color = [0] * n
    parent = [-1] * n
    for s0 in range(n):
        if color[s0]:
            continue
        stack = [(s0, 0)]
        color[s0] = 1
        while stack:
            x, it = stack[-1]
            if it < len(adj[x]):
                stack[-1] = (x, it + 1)
                y = adj[x][it]
                if color[y] == 0:
                    color[y] = 1
                    parent[y] = x
                    stack.append((y, 0))
                elif color[y] == 1:
                    cyc = [y]
                    z = x
                    while z != y:
                        cyc.append(z)
                        z = parent[z]
                    cyc.reverse()
                    pairs = list(zip(cyc, cyc[1:] + cyc[:1]))
                    viol = [data[p] for p in pairs if p in data]
                    return viol or [("cycle",)]
            else:
                color[x] = 2
                stack.pop()
    return []


def llm_subsequence(ops):
    name = {v: k for k, v in LLM_KIND.items()}
    return [(name[o.kind], o.mb, o.chunk) for o in ops if o.kind in name]


def peak_window(ops, open_kind, close_kind) -> int:
    cur = best = 0
    for o in ops:
        if o.kind == open_kind:
            cur += 1
            best = max(best, cur)
        elif o.kind == close_kind:
            cur -= 1
    return best


def order_property(cfg: SchedCfg, ops0):
    """Per unit i: (F_i, F_{i+1}, F_{i+2} precede G_i, G_i precedes F_{i+3})
    on the rank-0 list.  Returns list of (i, holds) for i+3 < n_u."""
    P = cfg.stages
    n_u = cfg.microbatches // P
    pos = {}
    for i, o in enumerate(ops0):
        if o.kind in (LLM_FWD, LLM_BWD):
            pos[(o.kind, o.mb, o.chunk)] = i
    F = [pos[(LLM_FWD, u * P, 0)] for u in range(n_u)]
    G = [pos[(LLM_BWD, u * P + P - 1, 0)] for u in range(n_u)]
    res = []
    for i in range(n_u - 3):
        res.append((i, F[i] < G[i] and F[i + 1] < G[i] and F[i + 2] < G[i] and G[i] < F[i + 3]))
    return res


# ----------------------------------------------------------------------------
# driver: the paper's train_step scheduler half
# ----------------------------------------------------------------------------
def build(cfg: SchedCfg) -> Schedule:
    validate(cfg)
    if cfg.llm_cp > 1 or cfg.enc_cp > 1:
        return build_cp(cfg)
    P, M, V = cfg.stages, cfg.microbatches, cfg.vchunks
    if cfg.llm_sched == "zb_h1":
        cw = wgrad_cost(cfg)
        cb = cfg.cost_bwd - cw
        base = zb_h1_schedule(P, M, cfg.cost_fwd, cb, cw)
    else:
        cw, cb = 0, cfg.cost_bwd
        base = llm_base_schedule(P, M, V)
    times = des_llm(base, P, V, cfg.cost_fwd, cb, cw)
    lists, W = nest(cfg, base, times)
    viol = verify_dependencies(cfg, lists)
    if viol:
        raise ScheduleError(E_DEPENDENCY, f"dependency violation: {viol[:3]}")
    for r in range(P):
        if llm_subsequence(lists[r]) != [tuple(x) for x in base[r]]:
            raise ScheduleError(E_DEPENDENCY, f"LLM order changed on rank {r}")
    with_comm, counts = insert_comm(cfg, lists)
    rings = size_rings(cfg, with_comm, counts)
    final = assign_slots(with_comm, rings)

    makespan = max(en for (_, en) in times.values())
    ws = w_star(base[0], P) if cfg.enc_place == "dp_unit" else 0
    stats = []
    for r in range(P):
        busy = sum(en - st for (rr, *_), (st, en) in times.items() if rr == r)
        rs = {p: 0 for p in PAYLOADS}
        for (src, dst, p), K in rings.items():
            if dst == r:
                rs[p] = max(rs[p], K)
        # a microbatch's stage activations live from F until B (until W under zb_h1)
        close = LLM_W if cfg.llm_sched == "zb_h1" else LLM_BWD
        inflight = cur = 0
        for o in lists[r]:
            if o.kind == LLM_FWD:
                cur += 1
                inflight = max(inflight, cur)
            elif o.kind == close:
                cur -= 1
        stats.append(Stats(
            w_star=ws, warmup_units=W if cfg.enc_place == "dp_unit" else 0,
            peak_enc_units=peak_window(lists[r], ENC_FWD, ENC_BWD),
            peak_gen_shards=peak_window(lists[r], GEN_FWD, GEN_BWD),
            peak_llm_inflight=inflight,
            llm_idle_cost_units=makespan - busy,
            makespan_cost_units=makespan,
            n_ops=len(final[r]),
            ring_slots=rs))
    return Schedule(cfg=cfg, ranks=final, stats=stats, rings=rings, llm_base=base, times=times)


# ----------------------------------------------------------------------------
# serialization (extends S:99 / S:274)
# ----------------------------------------------------------------------------
def _f(x):
    return "-" if (x is None or x == -1 or x == "") else str(x)


def serialize(sched: Schedule) -> str:
    lines = []
    for r, ops in enumerate(sched.ranks):
        for i, o in enumerate(ops):
            lines.append("\t".join([str(r), str(i), o.kind, _f(o.mb), _f(o.chunk), _f(o.unit),
                                    _f(o.peer), _f(o.payload), _f(o.slot), _f(o.seq)]))
    return "\n".join(lines) + ("\n" if lines else "")


# ----------------------------------------------------------------------------
# decoupled context parallelism (reading R25)
# ----------------------------------------------------------------------------
# R = P * llm_cp ranks, rank k = c P + r (LLM CP index c, pipeline stage r): the
# llm_cp ranks of a stage run the stage's LLM list in lockstep, each on its
# sequence shard of every microbatch.  The encoder runs in CP groups of enc_cp
# consecutive ranks, one microbatch per group, so an encoder unit has
# U = P llm_cp / enc_cp microbatches: microbatch uU + e on group e.  The
# encoder-to-LLM handoff is the CP-conversion all-to-all, expanded
# into P2P messages: every rank of m's encoder group sends "emb" to every
# stage-0 rank (c P) and receives "embgrad" back from each.  The generator runs
# on the last-stage ranks on their own rows (gen_place last_stage) or not at all.
def _stage_lists_and_times(cfg):
    P, M, V = cfg.stages, cfg.microbatches, cfg.vchunks
    if cfg.llm_sched == "zb_h1":
        cw = wgrad_cost(cfg)
        cb = cfg.cost_bwd - cw
        base = zb_h1_schedule(P, M, cfg.cost_fwd, cb, cw)
    else:
        cw, cb = 0, cfg.cost_bwd
        base = llm_base_schedule(P, M, V)
    return base, des_llm(base, P, V, cfg.cost_fwd, cb, cw)


def cp_encoder_ranks(cfg: SchedCfg, m: int):
    """Ranks of microbatch m's encoder CP group."""
    U = cfg.stages * cfg.llm_cp // cfg.enc_cp
    e = m % U
    return list(range(e * cfg.enc_cp, (e + 1) * cfg.enc_cp))


def cp_stage0_ranks(cfg: SchedCfg):
    return [c * cfg.stages for c in range(cfg.llm_cp)]


def _nest_cp(cfg, base, times):
    P, M, V = cfg.stages, cfg.microbatches, cfg.vchunks
    R, U = P * cfg.llm_cp, P * cfg.llm_cp // cfg.enc_cp
    n_u = M // U
    enc = cfg.enc_place == "dp_unit"
    W = (cfg.warmup_units if cfg.warmup_units > 0 else w_star(base[0], U)) if enc else 0
    events = []
    for k in range(R):
        for (kd, m, c) in base[k % P]:
            st, _ = times[(k % P, kd, m, c)]
            events.append((st, 2, k, (k, kd, m, c)))
    if cfg.gen_place != "none":
        for m in range(M):
            _, en = times[(P - 1, "F", m, V - 1)]
            events.append((en, 0, m, ("GEN", m)))
    if enc:
        for u in range(n_u):
            _, en = times[(0, "B", u * U + U - 1, 0)]
            events.append((en, 1, u, ("ENC", u)))
    events.sort(key=lambda e: (e[0], e[1], e[2]))
    lists = [[] for _ in range(R)]

    def unit_ops(kind, u):
        for k in range(R):
            for m in range(u * U, u * U + U):
                if k in cp_encoder_ranks(cfg, m):
                    lists[k].append(Op(kind, mb=m, unit=u))
    nxt = 0
    if enc:
        for u in range(min(W, n_u)):
            unit_ops(ENC_FWD, u)
        nxt = min(W, n_u)
    for _, cls, _, ev in events:
        if cls == 2:
            k, kd, m, c = ev
            if enc and kd == "F" and k % P == 0 and c == 0 and m // U >= nxt:
                raise ScheduleError(E_WARMUP, f"W={W} too small: F({m},0)@{k} precedes EncFwd({m // U})")
            lists[k].append(Op(LLM_KIND[kd], mb=m, chunk=c))
        elif cls == 0:
            m = ev[1]
            for c in range(cfg.llm_cp):
                lists[c * P + P - 1].append(Op(GEN_FWD, mb=m))
                lists[c * P + P - 1].append(Op(GEN_BWD, mb=m))
        else:
            u = ev[1]
            unit_ops(ENC_BWD, u)
            if nxt < n_u:
                unit_ops(ENC_FWD, nxt)
                nxt += 1
    return lists, W


def _cp_comm(cfg, k, op):
    """(recvs before, sends after) of compute op `op` on rank k."""
    P, V = cfg.stages, cfg.vchunks
    c, r = divmod(k, P)
    enc = cfg.enc_place == "dp_unit"
    before, after = [], []
    if op.kind in (LLM_FWD, LLM_BWD):
        s = vstage(P, r, op.chunk)
    if op.kind == LLM_FWD:
        if s > 0 and (s - 1) % P != r:
            before.append(Op(RECV, mb=op.mb, chunk=op.chunk, peer=c * P + (s - 1) % P, payload="act"))
        if s == 0 and enc:
            for q in cp_encoder_ranks(cfg, op.mb):
                if q != k:
                    before.append(Op(RECV, mb=op.mb, unit=op.mb // (P * cfg.llm_cp // cfg.enc_cp), peer=q,
                                     payload="emb"))
        if s < P * V - 1 and (s + 1) % P != r:
            after.append(Op(SEND, mb=op.mb, chunk=op.chunk, peer=c * P + (s + 1) % P, payload="act"))
    elif op.kind == LLM_BWD:
        if s < P * V - 1 and (s + 1) % P != r:
            before.append(Op(RECV, mb=op.mb, chunk=op.chunk, peer=c * P + (s + 1) % P, payload="grad"))
        if s > 0 and (s - 1) % P != r:
            after.append(Op(SEND, mb=op.mb, chunk=op.chunk, peer=c * P + (s - 1) % P, payload="grad"))
        if s == 0 and enc:
            for q in cp_encoder_ranks(cfg, op.mb):
                if q != k:
                    after.append(Op(SEND, mb=op.mb, unit=op.mb // (P * cfg.llm_cp // cfg.enc_cp), peer=q,
                                    payload="embgrad"))
    elif op.kind == ENC_FWD and enc:
        for q in cp_stage0_ranks(cfg):
            if q != k:
                after.append(Op(SEND, mb=op.mb, unit=op.unit, peer=q, payload="emb"))
    elif op.kind == ENC_BWD and enc:
        for q in cp_stage0_ranks(cfg):
            if q != k:
                before.append(Op(RECV, mb=op.mb, unit=op.unit, peer=q, payload="embgrad"))
    return before, after


def _cp_deps(cfg, k, op):
    P, V = cfg.stages, cfg.vchunks
    c, r = divmod(k, P)
    deps = []
    if op.kind in (LLM_FWD, LLM_BWD, LLM_W):
        s = vstage(P, r, op.chunk)
    if op.kind == LLM_FWD:
        if s > 0:
            deps.append((c * P + (s - 1) % P, LLM_FWD, op.mb, (s - 1) // P))
        elif cfg.enc_place == "dp_unit":
            deps += [(q, ENC_FWD, op.mb, -1) for q in cp_encoder_ranks(cfg, op.mb)]
    elif op.kind == LLM_BWD:
        deps.append((k, LLM_FWD, op.mb, op.chunk))
        if s < P * V - 1:
            deps.append((c * P + (s + 1) % P, LLM_BWD, op.mb, (s + 1) // P))
        elif cfg.gen_place == "last_stage":
            deps.append((k, GEN_BWD, op.mb, -1))
    elif op.kind == LLM_W:
        deps.append((k, LLM_BWD, op.mb, op.chunk))
    elif op.kind == ENC_BWD:
        deps.append((k, ENC_FWD, op.mb, -1))
        deps += [(q, LLM_BWD, op.mb, 0) for q in cp_stage0_ranks(cfg)]
    elif op.kind == GEN_FWD:
        deps.append((k, LLM_FWD, op.mb, V - 1))
    elif op.kind == GEN_BWD:
        deps.append((k, GEN_FWD, op.mb, -1))
    return deps


def _verify_with(lists, deps_fn):
    """verify_dependencies with a given producer function (acyclic program order + data)."""
    nid, n = {}, 0
    comp = [[op for op in ops if op.kind in COMPUTE_KINDS] for ops in lists]
    for k, ops in enumerate(comp):
        for op in ops:
            key = _ckey(k, op)
            if key in nid:
                return [("duplicate", key)]
            nid[key] = n
            n += 1
    edges = []
    for k, ops in enumerate(comp):
        for i, op in enumerate(ops):
            if i:
                edges.append((nid[_ckey(k, ops[i - 1])], nid[_ckey(k, op)]))
            for d in deps_fn(k, op):
                if d not in nid:
                    return [("missing", d, _ckey(k, op))]
                edges.append((nid[d], nid[_ckey(k, op)]))
    return [] if _acyclic(n, edges) else [("cycle",)]


def build_cp(cfg: SchedCfg) -> Schedule:
    """build() for decoupled CP (R25): nesting over P llm_cp ranks with encoder units of
    P llm_cp / enc_cp microbatches, CP-conversion messages, rings, verification."""
    P = cfg.stages
    R, U = P * cfg.llm_cp, P * cfg.llm_cp // cfg.enc_cp
    base, times = _stage_lists_and_times(cfg)
    lists, W = _nest_cp(cfg, base, times)
    viol = _verify_with(lists, lambda k, op: _cp_deps(cfg, k, op))
    if viol:
        raise ScheduleError(E_DEPENDENCY, f"dependency violation: {viol[:3]}")
    for k in range(R):
        if llm_subsequence(lists[k]) != [tuple(x) for x in base[k % P]]:
            raise ScheduleError(E_DEPENDENCY, f"LLM order changed on rank {k}")
    full = []
    for k in range(R):
        ops = []
        for op in lists[k]:
            before, after = _cp_comm(cfg, k, op)
            ops += before + [op] + after
        full.append(ops)
    send_cnt, recv_cnt = {}, {}
    for k in range(R):
        for i, op in enumerate(full[k]):
            if op.kind == SEND:
                ch = (k, op.peer, op.payload)
                full[k][i] = _with(op, seq=send_cnt.get(ch, 0))
                send_cnt[ch] = send_cnt.get(ch, 0) + 1
            elif op.kind == RECV:
                ch = (op.peer, k, op.payload)
                full[k][i] = _with(op, seq=recv_cnt.get(ch, 0))
                recv_cnt[ch] = recv_cnt.get(ch, 0) + 1
    if send_cnt != recv_cnt:
        raise ScheduleError(E_DEPENDENCY, "unmatched send/recv counts")
    rings = size_rings(cfg, full, send_cnt)
    final = assign_slots(full, rings)
    makespan = max(en for (_, en) in times.values())
    enc = cfg.enc_place == "dp_unit"
    ws = w_star(base[0], U) if enc else 0
    close = LLM_W if cfg.llm_sched == "zb_h1" else LLM_BWD
    stats = []
    for k in range(R):
        busy = sum(en - st for (rr, *_), (st, en) in times.items() if rr == k % P)
        rs = {p: 0 for p in PAYLOADS}
        for (src, dst, p), K in rings.items():
            if dst == k:
                rs[p] = max(rs[p], K)
        inflight = cur = 0
        for o in lists[k]:
            if o.kind == LLM_FWD:
                cur += 1
                inflight = max(inflight, cur)
            elif o.kind == close:
                cur -= 1
        stats.append(Stats(
            w_star=ws, warmup_units=W if enc else 0,
            peak_enc_units=peak_window(lists[k], ENC_FWD, ENC_BWD),
            peak_gen_shards=peak_window(lists[k], GEN_FWD, GEN_BWD),
            peak_llm_inflight=inflight,
            llm_idle_cost_units=makespan - busy,
            makespan_cost_units=makespan,
            n_ops=len(final[k]),
            ring_slots=rs))
    return Schedule(cfg=cfg, ranks=final, stats=stats, rings=rings, llm_base=[base[k % P] for k in range(R)],
                    times=times)
