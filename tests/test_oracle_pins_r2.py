"""Independent pins for the schedule oracle (round 2): each test re-derives its
expected value with machinery written here, never with oracle/schedule.py's own
graph, ring or DES helpers.

* ring sizing (P:317 deadlock_check): a token-game executor
  model written here (eager push into K receive slots, a slot freed after the
  op that consumes it) shows the oracle's rings are deadlock-free and minimal,
  and reproduces SURVEY A4's independently computed sizes under the stash rule;
* compute optimality: exhaustive search over
  every full-width cut placement of the encoder units finds no shorter makespan
  than BigMac's, and exhaustive free per-rank placement shows the documented
  12 vs 14 gap at P = 2, M = 4;
* reading R2 (P:198 vs P:211-212): a generator unit of P microbatches has no
  legal placement on any rank (brute force), while per-microbatch shards do;
* interleaved 1F1B peak in-flight min(w_r + 1, MV) (Narayanan et al.'s
  warmup);
* the fp64 schedule interpreter (bounded receive slots) on the C2, C3 and C4
  schedule shapes.
"""
import itertools

import numpy as np
import pytest

from oracle import schedule as S


def cfg_of(P, M, V, **kw):
    return S.SchedCfg(P, M, V, llm_sched="1f1b" if V == 1 else "interleaved", **kw)


# =========================================================================== rings
def _consumer(ops, i, rule):
    """Index of the op after which the message received at ops[i] is freed."""
    o = ops[i]
    if rule == "stash" and o.payload == "act":
        # SURVEY A4 scratch rule: the act slot doubles as the stage-input stash,
        # freed by the receiver's backward of the same (mb, chunk)
        j = i + 1
        while not (ops[j].kind == "LlmBwd" and ops[j].mb == o.mb and ops[j].chunk == o.chunk):
            j += 1
        return j
    j = i + 1
    while ops[j].kind in ("Send", "Recv"):
        j += 1
    if o.payload == "genin":   # read by GenFwd and GenBwd (the executor's reading R6)
        while ops[j].kind != "GenBwd":
            j += 1
    return j


def token_game(ranks, K, rule="consumer"):
    """Run the executor model with K[(src, dst, payload)] receive slots per channel
    and zero durations.  Per rank: a program-order stream of every non-Send op
    (Recv waits for its message), and one stream per peer for its Sends (a Send
    waits for the op before it in program order -- its producer -- and for a
    free slot: message j may be pushed once message j - K has been consumed).
    Returns True iff every op fires (no deadlock)."""
    P = len(ranks)
    sends, recv_of, freed_by = {}, {}, {}
    for r, ops in enumerate(ranks):
        for i, o in enumerate(ops):
            if o.kind == "Send":
                sends[((r, o.peer, o.payload), o.seq)] = (r, i)
            elif o.kind == "Recv":
                ch = (o.peer, r, o.payload)
                recv_of[(r, i)] = (ch, o.seq)
                freed_by[(ch, o.seq)] = (r, _consumer(ops, i, rule))
    done = set()
    main = [0] * P                                   # next non-Send op per rank
    sq = [{} for _ in range(P)]                      # peer -> next send index
    send_lists = [{} for _ in range(P)]
    producer = {}
    for r, ops in enumerate(ranks):
        last = None
        for i, o in enumerate(ops):
            if o.kind == "Send":
                send_lists[r].setdefault(o.peer, []).append(i)
                producer[(r, i)] = last
            else:
                last = i
        for q in send_lists[r]:
            sq[r][q] = 0
    total = sum(len(x) for x in ranks)
    progress = True
    while progress:
        progress = False
        for r, ops in enumerate(ranks):
            # main stream
            while True:
                i = main[r]
                while i < len(ops) and ops[i].kind == "Send":
                    i += 1
                main[r] = i
                if i >= len(ops):
                    break
                if ops[i].kind == "Recv":
                    ch, seq = recv_of[(r, i)]
                    if sends[(ch, seq)] not in done:
                        break
                done.add((r, i))
                main[r] = i + 1
                progress = True
            # send streams
            for q, lst in send_lists[r].items():
                while sq[r][q] < len(lst):
                    i = lst[sq[r][q]]
                    o = ops[i]
                    p = producer[(r, i)]
                    if p is not None and (r, p) not in done:
                        break
                    ch = (r, o.peer, o.payload)
                    k = K[ch]
                    if o.seq >= k and freed_by[(ch, o.seq - k)] not in done:
                        break
                    done.add((r, i))
                    sq[r][q] += 1
                    progress = True
    return len(done) == total


def _channels(ranks):
    cnt = {}
    for r, ops in enumerate(ranks):
        for o in ops:
            if o.kind == "Send":
                cnt[(r, o.peer, o.payload)] = cnt.get((r, o.peer, o.payload), 0) + 1
    return cnt


def _min_k(ranks, cnt, ch, rule):
    """Smallest K on `ch` (all other channels unbounded) that completes; binary
    search (more slots never hurt)."""
    K = dict(cnt)
    lo, hi = 1, cnt[ch]
    while lo < hi:
        mid = (lo + hi) // 2
        K[ch] = mid
        if token_game(ranks, K, rule):
            hi = mid
        else:
            lo = mid + 1
    return lo


@pytest.mark.parametrize("P,M,V", [(2, 4, 1), (4, 16, 1), (4, 32, 2), (8, 64, 1), (2, 8, 2)])
def test_oracle_rings_deadlock_free_and_minimal_independent(P, M, V):
    # the oracle's rings (no slack) complete under the executor model written
    # here; every channel with K > 1 deadlocks with one slot fewer
    s = S.build(cfg_of(P, M, V, ring_slack=0))
    assert token_game(s.ranks, s.rings)
    for ch, k in s.rings.items():
        if k > 1:
            K = dict(s.rings)
            K[ch] = k - 1
            assert not token_game(s.ranks, K), ch


def test_token_game_detects_slot_starvation():
    # the model is not vacuous: when act slots are held until the receiver's backward
    # (stash rule), one slot per channel starves the 1F1B warmup and must deadlock
    s = S.build(cfg_of(4, 16, 1, ring_slack=0))
    K = {ch: 1 for ch in _channels(s.ranks)}
    assert not token_game(s.ranks, K, rule="stash")


@pytest.mark.parametrize("P,M,V,W,act", [(4, 16, 1, 3, 3), (8, 64, 1, 3, 7), (4, 32, 2, 3, 13), (8, 64, 2, 3, 29)])
def test_survey_ring_sizes_under_stash_rule(P, M, V, W, act):
    # SURVEY §8(a) A4 / Appendix A.5 (computed at survey time with throwaway scripts):
    # act slots doubling as the stage-input stash need 13 (P=4, V=2) / 29 (P=8, V=2)
    # slots; grad <= 4; emb 2; embgrad, genin, gengrad 1 -- all reproduced here.  For
    # 1F1B the survey wrote "act = P"; the busiest act channel (0 -> 1) feeds rank 1,
    # whose 1F1B in-flight depth is P - 1 (textbook min(P - r, M) at r = 1), so P - 1
    # slots suffice and are necessary (reading R17)
    s = S.build(cfg_of(P, M, V, warmup_units=W, ring_slack=0))
    cnt = _channels(s.ranks)
    need = {}
    for ch in cnt:
        k = _min_k(s.ranks, cnt, ch, "stash")
        need[ch[2]] = max(need.get(ch[2], 0), k)
    assert need["act"] == act
    assert need["grad"] <= 4
    assert need["emb"] == 2
    assert need["embgrad"] == need["genin"] == need["gengrad"] == 1


# =========================================================================== compute optimality
def _vst(P, r, c):
    return c * P + r


def des(P, V, lists, cost):
    """Independent compute-only DES (zero-latency comm): each rank runs its list in
    order, an op starts at max(end of its predecessor on the rank, end of its data
    producers).  Producers: F(m, s-1); B(m, s+1) and F(m, s); the encoder unit's
    EncFwd for F(m, 0); B(m, 0) for EncBwd.  Returns the makespan or None on a
    dependency deadlock."""
    PV = P * V
    key_rank = {}
    for r, ops in enumerate(lists):
        for o in ops:
            key_rank[_k(o, r, P)] = r
    end = {}
    ptr = [0] * P
    clock = [0] * P
    n = sum(len(x) for x in lists)
    fired = 0
    while fired < n:
        moved = False
        for r, ops in enumerate(lists):
            while ptr[r] < len(ops):
                o = ops[ptr[r]]
                deps = _deps(o, r, P, V, PV)
                if any(d not in end for d in deps):
                    break
                t0 = max([clock[r]] + [end[d] for d in deps])
                t1 = t0 + cost(o)
                end[_k(o, r, P)] = t1
                clock[r] = t1
                ptr[r] += 1
                fired += 1
                moved = True
        if not moved:
            return None
    return max(clock)


def _k(o, r, P):
    if o.kind in ("LlmFwd", "LlmBwd"):
        return (o.kind, o.mb, _vst(P, r, o.chunk))
    if o.kind in ("EncFwd", "EncBwd"):
        return (o.kind, o.unit, r)
    return (o.kind, o.mb, r)


def _deps(o, r, P, V, PV):
    if o.kind == "LlmFwd":
        s = _vst(P, r, o.chunk)
        if s > 0:
            return [("LlmFwd", o.mb, s - 1)]
        return [("EncFwd", o.mb // P, o.mb % P)]
    if o.kind == "LlmBwd":
        s = _vst(P, r, o.chunk)
        d = [("LlmFwd", o.mb, s)]
        if s < PV - 1:
            d.append(("LlmBwd", o.mb, s + 1))
        return d
    if o.kind == "EncBwd":
        return [("LlmBwd", o.unit * P + r, 0)]
    return []


def _llm_ops(P, M, V, r):
    return [S.Op("LlmFwd" if k == "F" else "LlmBwd", mb=m, chunk=c) for k, m, c in S.llm_base_schedule(P, M, V)[r]]


def _cut_times(P, M, V, cf, cb):
    """Start times of every LLM op in the cut timeline (1F1B DES, costs cf / cb),
    computed here from the base lists with the DES above."""
    lists = [_llm_ops(P, M, V, r) for r in range(P)]
    starts = [[] for _ in range(P)]
    end = {}
    ptr, clock = [0] * P, [0] * P
    PV = P * V
    n = sum(len(x) for x in lists)
    fired = 0
    while fired < n:
        for r, ops in enumerate(lists):
            while ptr[r] < len(ops):
                o = ops[ptr[r]]
                deps = [d for d in _deps(o, r, P, V, PV) if d[0] != "EncFwd"]
                if any(d not in end for d in deps):
                    break
                t0 = max([clock[r]] + [end[d] for d in deps])
                starts[r].append(t0)
                end[_k(o, r, P)] = t0 + (cf if o.kind == "LlmFwd" else cb)
                clock[r] = end[_k(o, r, P)]
                ptr[r] += 1
                fired += 1
    return lists, starts, max(clock)


def cut_class_min(P, M, cf, cb, ef, eb):
    """Minimum makespan over every full-width cut placement of the n_u encoder units
    (V = 1): EncFwd(u) / EncBwd(u) inserted on every rank before all LLM ops whose
    cut-timeline start is >= its cut time; units in order within a kind; at equal
    cut times backward before forward, then by unit."""
    lists, starts, mk = _cut_times(P, M, 1, cf, cb)
    taus = sorted({t for st in starts for t in st} | {mk})
    n_u = M // P
    best = None

    def cost(o):
        return {"LlmFwd": cf, "LlmBwd": cb, "EncFwd": ef, "EncBwd": eb}[o.kind]
    for tf in itertools.combinations_with_replacement(taus, n_u):
        for tb in itertools.combinations_with_replacement(taus, n_u):
            ins = [(t, 1, u, "EncFwd") for u, t in enumerate(tf)] + [(t, 0, u, "EncBwd") for u, t in enumerate(tb)]
            ins.sort()
            out = []
            for r in range(P):
                merged, k = [], 0
                for o, t0 in zip(lists[r], starts[r]):
                    while k < len(ins) and ins[k][0] <= t0:
                        merged.append(S.Op(ins[k][3], mb=ins[k][2] * P + r, unit=ins[k][2]))
                        k += 1
                    merged.append(o)
                merged += [S.Op(x[3], mb=x[2] * P + r, unit=x[2]) for x in ins[k:]]
                out.append(merged)
            if not _enc_fifo_ok(out[0]):
                continue
            m = des(P, 1, out, cost)
            if m is not None and (best is None or m < best):
                best = m
    return best


def _enc_fifo_ok(ops):
    live = set()
    for o in ops:
        if o.kind == "EncFwd":
            live.add(o.unit)
        elif o.kind == "EncBwd":
            if o.unit not in live:
                return False
    return True


def bigmac_makespan(P, M, cf, cb, ef, eb):
    s = S.build(cfg_of(P, M, 1, gen_place="none", cost_fwd=cf, cost_bwd=cb))
    lists = [[o for o in ops if o.kind in S.COMPUTE_KINDS] for ops in s.ranks]
    return des(P, 1, lists, lambda o: {"LlmFwd": cf, "LlmBwd": cb, "EncFwd": ef, "EncBwd": eb}[o.kind])


def ce_makespan(P, M, cf, cb, ef, eb):
    """The compute-efficient design: every EncFwd first (W = n_u)."""
    s = S.build(cfg_of(P, M, 1, gen_place="none", cost_fwd=cf, cost_bwd=cb, warmup_units=M // P))
    lists = [[o for o in ops if o.kind in S.COMPUTE_KINDS] for ops in s.ranks]
    return des(P, 1, lists, lambda o: {"LlmFwd": cf, "LlmBwd": cb, "EncFwd": ef, "EncBwd": eb}[o.kind])


@pytest.mark.parametrize("P,M,cf,cb,ef,eb", [(2, 4, 1, 1, 1, 1), (2, 4, 1, 2, 1, 2), (3, 6, 1, 1, 1, 1),
                                             (3, 6, 1, 2, 1, 2), (2, 6, 1, 2, 1, 1), (4, 8, 1, 2, 1, 2),
                                             (4, 16, 2, 4, 1, 2), (8, 16, 1, 2, 1, 1)])
def test_bigmac_matches_compute_efficient(P, M, cf, cb, ef, eb):
    # P:45 ("the same computational efficiency as the compute-efficient design") and
    # under the independent DES BigMac's makespan equals the compute-efficient
    # pipeline's, T_LLM + n_u (ef + eb) with T_LLM = (M + P - 1)(cf + cb) --
    # the nested units cost exactly their own work, while holding W* units, not M / P
    bm = bigmac_makespan(P, M, cf, cb, ef, eb)
    assert bm == ce_makespan(P, M, cf, cb, ef, eb)
    assert bm == (M + P - 1) * (cf + cb) + (M // P) * (ef + eb)
    # every full-width cut placement is at most that long (an inserted node delays the
    # ops after its cut by at most its own length -- the argument behind reading R1)
    if M // P <= 2 and P <= 3:
        assert cut_class_min(P, M, cf, cb, ef, eb) <= bm


def free_placement_min(P, M, cf, cb, ef, eb):
    """Exhaustive minimum over EVERY per-rank insertion of EncFwd(u)/EncBwd(u)
    (u in order within a kind, EncBwd(u) after EncFwd(u)) into each rank's LLM list."""
    n_u = M // P
    llm = [_llm_ops(P, M, 1, r) for r in range(P)]

    def orders():
        out = []

        def rec(nf, nb, acc):
            if nf == n_u and nb == n_u:
                out.append(list(acc))
                return
            if nf < n_u:
                rec(nf + 1, nb, acc + [("EncFwd", nf)])
            if nb < nf:
                rec(nf, nb + 1, acc + [("EncBwd", nb)])
        rec(0, 0, [])
        return out

    def placements(r):
        L = len(llm[r])
        res = []
        for slots in itertools.combinations(range(L + 2 * n_u), 2 * n_u):
            for od in orders():
                merged, li, ei = [], 0, 0
                sset = set(slots)
                for p in range(L + 2 * n_u):
                    if p in sset:
                        k, u = od[ei]
                        merged.append(S.Op(k, mb=u * P + r, unit=u))
                        ei += 1
                    else:
                        merged.append(llm[r][li])
                        li += 1
                res.append(merged)
        return res

    def cost(o):
        return {"LlmFwd": cf, "LlmBwd": cb, "EncFwd": ef, "EncBwd": eb}[o.kind]
    per = [placements(r) for r in range(P)]
    best = None
    for combo in itertools.product(*per):
        m = des(P, 1, list(combo), cost)
        if m is not None and (best is None or m < best):
            best = m
    return best


def test_free_placement_gap_p2_m4():
    # over ALL per-rank placements (exhaustive, no
    # cut restriction) the minimum at P = 2, M = 4, unit costs is 12 -- fill/drain
    # bubbles can absorb encoder work -- while BigMac and compute-efficient give 14.
    # Cut placements that park an EncFwd / EncBwd in a rank's fill or drain idle time
    # reach 12 as well, so the paper's claim (BigMac = compute-efficient time)
    # holds, and optimality against all placements does not (reading R18)
    assert free_placement_min(2, 4, 1, 1, 1, 1) == 12
    assert bigmac_makespan(2, 4, 1, 1, 1, 1) == ce_makespan(2, 4, 1, 1, 1, 1) == 14
    assert cut_class_min(2, 4, 1, 1, 1, 1) == 12


# =========================================================================== reading R2
def _gen_unit_feasible(P, M, V, r, i, j, unit_mbs):
    """Is there a legal execution with GenFwd(U)/GenBwd(U) of one generator unit
    inserted at positions i <= j of rank r's LLM list?  GenFwd needs every
    F(m, V-1) of the unit (last virtual stage, rank P-1); GenBwd needs GenFwd; each
    B(m, V-1) of the unit needs GenBwd (its input gradient)."""
    lists = [_llm_ops(P, M, V, q) for q in range(P)]
    gf, gb = S.Op("GenFwd", mb=-1), S.Op("GenBwd", mb=-2)
    lst = list(lists[r])
    lst.insert(j, gb)
    lst.insert(i, gf)
    lists[r] = lst
    PV = P * V
    end, ptr = set(), [0] * P
    n = sum(len(x) for x in lists)
    fired = 0
    while fired < n:
        moved = False
        for q, ops in enumerate(lists):
            while ptr[q] < len(ops):
                o = ops[ptr[q]]
                if o.kind == "GenFwd":
                    deps = [("LlmFwd", m, PV - 1) for m in unit_mbs]
                elif o.kind == "GenBwd":
                    deps = [("GenFwd",)]
                else:
                    deps = [d for d in _deps(o, q, P, V, PV) if d[0] != "EncFwd"]
                    if o.kind == "LlmBwd" and _vst(P, q, o.chunk) == PV - 1 and o.mb in unit_mbs:
                        deps.append(("GenBwd",))
                if any(d not in end for d in deps):
                    break
                end.add(("GenFwd",) if o.kind == "GenFwd" else ("GenBwd",) if o.kind == "GenBwd"
                        else _k(o, q, P))
                ptr[q] += 1
                fired += 1
                moved = True
        if not moved:
            return False
    return True


@pytest.mark.parametrize("P,M,V", [(2, 2, 1), (2, 4, 1), (3, 3, 1), (2, 4, 2), (3, 6, 2)])
def test_generator_unit_of_p_microbatches_infeasible(P, M, V):
    # DESIGN R2: a generator unit of P microbatches (P:198 read literally) has NO legal
    # placement -- brute force over every rank and every pair of insertion points --
    # because the last rank runs B(m, V-1) right after F(m, V-1); a per-microbatch
    # generator op (the reading taken) always has one
    for r in range(P):
        L = len(S.llm_base_schedule(P, M, V)[r])
        for i in range(L + 1):
            for j in range(i, L + 1):
                assert not _gen_unit_feasible(P, M, V, r, i, j, list(range(P)))
    ok = any(_gen_unit_feasible(P, M, V, P - 1, i, j, [0])
             for i in range(len(S.llm_base_schedule(P, M, V)[P - 1]) + 1)
             for j in range(i, len(S.llm_base_schedule(P, M, V)[P - 1]) + 1))
    assert ok


# =========================================================================== interleaved memory
@pytest.mark.parametrize("P,V,M", [(2, 2, 4), (2, 2, 8), (4, 2, 8), (4, 2, 32), (4, 4, 32), (8, 2, 64), (3, 3, 9)])
def test_interleaved_peak_inflight(P, V, M):
    # interleaved 1F1B (Narayanan et al.): rank r runs w_r = min(2(P-r-1) + (V-1)P, MV)
    # warmup forwards before its first backward, so it holds min(w_r + 1, MV) chunk
    # activations at peak
    s = S.build(cfg_of(P, M, V))
    for r in range(P):
        w = min(2 * (P - r - 1) + (V - 1) * P, M * V)
        assert s.stats[r].peak_llm_inflight == min(w + 1, M * V)


# =========================================================================== interpreter at bench shapes
@pytest.mark.parametrize("P,M,V,L", [(4, 16, 1, 4), (4, 32, 2, 8), (8, 64, 1, 8)])
def test_interpreter_on_bench_schedules(P, M, V, L):
    # the C2 (4 stages, 16 mb), C3 (4 stages, 32 mb, interleaved x2) and C4 (8 stages,
    # 64 mb) schedules -- tiny C1-sized blocks -- run in the fp64 interpreter with the
    # oracle's bounded receive rings (slot overwrite / buffer miss / leak raise) and
    # reach the sequential gradients
    from synth import get_config, make_batch, make_weights
    from oracle import interp
    from oracle import model as om
    cfg = get_config("C1", P=P, M=M, V=V).replace(L=L)
    if V > 1:
        cfg = cfg.replace(llm_sched="interleaved")
    W, B = make_weights(cfg), make_batch(cfg)
    loss, per, G = om.step_fp64(cfg, W, B)
    sched = S.build(S.SchedCfg(P, M, V, llm_sched=cfg.llm_sched))
    loss2, per2, G2, _ = interp.run(sched, cfg, W, B)
    assert abs(loss2 - loss) <= 1e-12 * abs(loss)
    for k in G:
        assert np.linalg.norm(G2[k] - G[k]) <= 1e-12 * max(np.linalg.norm(G[k]), 1e-30), k


# =========================================================================== degenerate batches
@pytest.mark.parametrize("P,M,V", [(1, 4, 1), (4, 4, 1), (2, 8, 2)])
def test_edge_batches_interpreter_and_closed_forms(P, M, V):
    # the method's degenerate microbatches (synth.edge_counts): n_mod = 0, n_mod = S (no
    # CE rows: CE_m = 0 by reading R8's mean over an empty set), generator rows covering
    # the whole sequence, n_gen < P (empty generator shards); the interpreter (per-rank
    # shards, gather / scatter of empty messages) equals the sequential definition
    from synth import edge_counts, edge_shape, get_config, make_batch, make_weights
    from oracle import interp
    from oracle import model as om
    cfg = edge_shape(get_config("C1", P=P, M=M, V=V))
    n_mod, n_gen = edge_counts(cfg, M)
    W, B = make_weights(cfg), make_batch(cfg, n_mod=n_mod, n_gen=n_gen)
    loss, per, G = om.step_fp64(cfg, W, B)
    for m in range(M):
        if n_mod[m] == cfg.S:
            assert per[m][0] == 0.0
    assert all(np.isfinite(v).all() for v in G.values())
    sched = S.build(S.SchedCfg(P, M, V, llm_sched=cfg.llm_sched))
    loss2, per2, G2, _ = interp.run(sched, cfg, W, B)
    assert abs(loss2 - loss) <= 1e-12 * abs(loss)
    for k in G:
        assert np.linalg.norm(G2[k] - G[k]) <= 1e-12 * max(np.linalg.norm(G[k]), 1e-30), k


def test_no_modality_rows_gives_zero_encoder_gradients():
    # with n_mod = 0 in every microbatch the encoder and projector never touch the loss:
    # their gradients are exactly zero (the embedding is all text rows)
    from synth import edge_shape, get_config, make_batch, make_weights
    from oracle import model as om
    cfg = edge_shape(get_config("C1", P=1, M=2))
    W, B = make_weights(cfg), make_batch(cfg, n_mod=[0, 0], n_gen=[5, 9])
    _, _, G = om.step_fp64(cfg, W, B)
    for k, v in G.items():
        if k.startswith("enc."):
            assert not np.any(v), k


# =========================================================================== reading R20
@pytest.mark.parametrize("parts", [[0, 40, 40, 97], [0, 97], [0, 0, 13, 97], [0, 30, 60, 97, 97]])
def test_generator_row_partition_invariance(parts):
    # R20: the generator is token-wise, so running it on any partition of a microbatch's
    # n_gen rows (empty parts included) with the full-microbatch MSE denominator and
    # summing the parts' losses and gradients gives the unsharded result (up to fp64
    # summation order) -- what gen_exclude relies on
    from synth import get_config, make_weights
    from oracle import model as om
    cfg = get_config("C1")
    W = om.to_f64(make_weights(cfg))
    rng = np.random.default_rng(7)
    n = parts[-1]
    X = rng.standard_normal((n, cfg.d))
    t = rng.standard_normal((n, cfg.d_t))
    denom = float(n * cfg.d_t)
    G_full = {}
    mse, cache = om.gen_fwd(W, cfg, X, t, denom)
    dX = om.gen_bwd(W, cfg, cache, 1.0, G_full)
    G_sum, mse_sum, dX_parts = {}, 0.0, []
    for a, b in zip(parts[:-1], parts[1:]):
        if b == a:
            continue
        m, c = om.gen_fwd(W, cfg, X[a:b], t[a:b], denom)
        mse_sum += m
        dX_parts.append(om.gen_bwd(W, cfg, c, 1.0, G_sum))
    assert abs(mse_sum - mse) <= 1e-12 * abs(mse)
    assert np.allclose(np.concatenate(dX_parts), dX, rtol=1e-12, atol=1e-15)
    for k in G_full:
        assert np.linalg.norm(G_sum[k] - G_full[k]) <= 1e-12 * np.linalg.norm(G_full[k]), k


# =========================================================================== reading R22
@pytest.mark.parametrize("P,M,V,ex", [(4, 16, 1, 4), (4, 8, 1, 1), (2, 4, 1, 2), (4, 16, 2, 4), (3, 6, 1, 3)])
def test_encoder_exclusion(P, M, V, ex):
    # R22: with ranks masked out of the encoder, every microbatch's EncFwd / EncBwd still
    # runs exactly once, on an unmasked rank (the nearest lower one, cyclically), in
    # microbatch order within a unit; the emb / embgrad messages follow the owner; the
    # nested schedule stays dependency-safe with the same W*; the interpreter reproduces
    # the sequential gradients
    from synth import get_config, make_batch, make_weights
    from oracle import interp
    from oracle import model as om
    sched = "1f1b" if V == 1 else "interleaved"
    s = S.build(cfg_of(P, M, V, enc_exclude=ex))
    plain = S.build(cfg_of(P, M, V))
    owner = {}
    for r, ops in enumerate(s.ranks):
        fw = [o.mb for o in ops if o.kind == "EncFwd"]
        assert fw == sorted(fw)
        for m in fw:
            assert m not in owner
            owner[m] = r
        if (ex >> r) & 1:
            assert not fw
    assert sorted(owner) == list(range(M))
    for m, r in owner.items():
        q = m % P
        while (ex >> q) & 1:
            q = (q - 1) % P
        assert r == q
    sends = {(o.mb, r) for r, ops in enumerate(s.ranks) for o in ops if o.kind == "Send" and o.payload == "emb"}
    assert sends == {(m, r) for m, r in owner.items() if r != 0}
    assert s.stats[0].w_star == plain.stats[0].w_star
    comp = [[o for o in ops if o.kind in S.COMPUTE_KINDS] for ops in s.ranks]
    assert S.verify_dependencies(s.cfg, comp) == []
    L = P * V if (P * V) % 2 == 0 or P * V > 2 else 2
    cfg = get_config("C1", P=P, M=M, V=V).replace(L=L, llm_sched=sched)
    W, B = make_weights(cfg), make_batch(cfg)
    loss, _, G = om.step_fp64(cfg, W, B)
    loss2, _, G2, _ = interp.run(s, cfg, W, B)
    assert abs(loss2 - loss) <= 1e-12 * abs(loss)
    for k in G:
        assert np.linalg.norm(G2[k] - G[k]) <= 1e-12 * max(np.linalg.norm(G[k]), 1e-30), k
