"""Pins for the schedule oracle (O-S) against what the paper and mathematics fix.

Each test names the passage it pins.  None of these retypes the oracle's own
construction: they check worked examples, closed forms
(P:162), invariants, brute force on tiny inputs, and
mutations that must be detected.
"""
import itertools

import pytest

from oracle import schedule as S
from oracle.bruteforce import min_peak_encoder_window
from oracle.des import simulate, uniform_cost


def cfg_of(P, M, V, **kw):
    return S.SchedCfg(P, M, V, llm_sched="1f1b" if V == 1 else "interleaved", **kw)


GRID = [(P, V, M) for P in (1, 2, 4, 8) for V in (1, 2, 4) for M in (P, 2 * P, 8 * P, 16 * P)
        if not (P == 8 and M == 16 * P and V == 4)]


# --------------------------------------------------------------------------- A1
def test_1f1b_single_stage_example():
    # (P=1, M=3) -> F0 B0 F1 B1 F2 B2
    assert S.llm_base_schedule(1, 3, 1)[0] == [("F", 0, 0), ("B", 0, 0), ("F", 1, 0),
                                               ("B", 1, 0), ("F", 2, 0), ("B", 2, 0)]


def test_1f1b_rank0_forwards_before_first_backward():
    # (P=4, M=8) -> rank 0 runs 4 forwards before its first backward
    ops = S.llm_base_schedule(4, 8, 1)[0]
    assert [k for k, _, _ in ops].index("B") == 4


def test_interleaved_rank0_warmup():
    # (P=4, V=2, M=8) -> rank 0 warmup = (P-1)*2 + (V-1)*P = 10 forwards
    ops = S.llm_base_schedule(4, 8, 2)[0]
    assert [k for k, _, _ in ops].index("B") == 11  # 10 warmup F + the first steady F
    # (P=4, V=2, M=64) -> 256 ops per rank
    assert all(len(l) == 256 for l in S.llm_base_schedule(4, 64, 2))


@pytest.mark.parametrize("P,V,M", GRID)
def test_base_schedule_complete_and_feasible(P, V, M):
    # every (mb, chunk) exactly once as F and as B per rank; dependency feasible
    base = S.llm_base_schedule(P, M, V)
    for ops in base:
        assert sorted(x for x in ops if x[0] == "F") == [("F", m, c) for m in range(M) for c in range(V)]
        assert sorted(x for x in ops if x[0] == "B") == [("B", m, c) for m in range(M) for c in range(V)]
        seen = set()
        for k, m, c in ops:  # forward precedes backward on the same rank
            if k == "B":
                assert (m, c) in seen
            seen.add((m, c))
    S.des_llm(base, P, V, 1, 2)  # raises on a dependency stall


@pytest.mark.parametrize("P,V,M", GRID)
@pytest.mark.parametrize("cf,cb", [(1, 1), (1, 2), (2, 3)])
def test_des_closed_form_bubble(P, V, M, cf, cb):
    # fill/drain overhead of 1F1B -> per-rank idle (P-1)(cf+cb), makespan (MV+P-1)(cf+cb)
    times = S.des_llm(S.llm_base_schedule(P, M, V), P, V, cf, cb)
    mk = max(e for _, e in times.values())
    assert mk == (M * V + P - 1) * (cf + cb)
    for r in range(P):
        busy = sum(e - s for (rr, *_), (s, e) in times.items() if rr == r)
        assert mk - busy == (P - 1) * (cf + cb)


def test_bubble_rate_paper_value():
    # P:162 / S:304 / S:548: 1F1B P=4, M=64, uniform costs -> bubble (P-1)/(M+P-1) = 3/67
    s = S.build(cfg_of(4, 64, 1, cost_fwd=1, cost_bwd=1))
    st = s.stats[3]
    assert abs(st.llm_idle_cost_units / st.makespan_cost_units - 3 / 67) < 1e-9


@pytest.mark.parametrize("P,M", [(2, 4), (4, 8), (4, 16), (8, 64)])
def test_1f1b_peak_inflight(P, M):
    # textbook 1F1B (Narayanan et al.): rank r holds at most min(P - r, M) activations
    s = S.build(cfg_of(P, M, 1))
    assert [st.peak_llm_inflight for st in s.stats] == [min(P - r, M) for r in range(P)]


# --------------------------------------------------------------------------- A3 nesting
def test_trivial_chain():
    # (P=1, M=1, W=1) -> EncFwd, LlmFwd, GenFwd, GenBwd, LlmBwd, EncBwd
    s = S.build(cfg_of(1, 1, 1, warmup_units=1))
    assert [o.kind for o in s.ranks[0]] == ["EncFwd", "LlmFwd", "GenFwd", "GenBwd", "LlmBwd", "EncBwd"]


@pytest.mark.parametrize("P,V,M", [g for g in GRID if g[2] % g[0] == 0])
def test_nesting_invariants(P, V, M):
    s = S.build(cfg_of(P, M, V))
    base = S.llm_base_schedule(P, M, V)
    W = s.stats[0].warmup_units
    for r in range(P):
        # P:209 / S:209: LLM order unchanged
        assert S.llm_subsequence(s.ranks[r]) == base[r]
        # P:212 / S:210-211: encoder window <= W, generator window <= 1
        assert s.stats[r].peak_enc_units <= W
        assert s.stats[r].peak_gen_shards == 1
    comp = [[o for o in ops if o.kind in S.COMPUTE_KINDS] for ops in s.ranks]
    assert S.verify_dependencies(s.cfg, comp) == []


@pytest.mark.parametrize("P,V,M", [(2, 1, 4), (2, 1, 8), (3, 1, 9), (2, 2, 8), (3, 2, 12), (4, 2, 16)])
def test_min_peak_bruteforce_equals_wstar(P, V, M):
    # earliest dependency-safe placement -> BigMac's window with W = W*
    # equals the minimum peak over ALL dependency-safe interleavings (brute force)
    s = S.build(cfg_of(P, M, V))
    assert s.stats[0].w_star == min_peak_encoder_window(P, M, V)
    assert s.stats[0].peak_enc_units == s.stats[0].w_star


def test_paper_fig4_setting():
    # P:180 Fig.4 (pp=4, vpp=2, batch 64), P:212/216/228: W = 3, peak live units 3 per rank
    s = S.build(cfg_of(4, 64, 2))
    assert s.stats[0].w_star == 3
    assert all(st.peak_enc_units == 3 for st in s.stats)
    assert all(st.peak_gen_shards == 1 for st in s.stats)
    assert M_units(s) == 16


def M_units(s):
    return len({o.unit for o in s.ranks[0] if o.kind == "EncFwd"})


@pytest.mark.parametrize("P,V,M", [(3, 2, 12), (4, 2, 32), (4, 2, 64), (8, 2, 64), (4, 4, 32), (3, 3, 18)])
def test_order_property_holds_p3_v2(P, V, M):
    # F_i, F_{i+1}, F_{i+2} < G_i < F_{i+3} for interleaved vpp >= 2
    s = S.build(cfg_of(P, M, V))
    res = S.order_property(s.cfg, s.ranks[0])
    assert res and all(ok for _, ok in res)


def test_order_property_fails_at_p2():
    # SPEC S:186 claims (P=2, V=2, M=16) passes; with the construction of P:200 it does
    # not (G_i precedes F_{i+2}) -- reading recorded in DESIGN.md.
    s = S.build(cfg_of(2, 16, 2))
    assert not all(ok for _, ok in S.order_property(s.cfg, s.ranks[0]))
    assert s.stats[0].w_star == 2


@pytest.mark.parametrize("P,V,M,w", [(1, 1, 4, 1), (2, 1, 8, 2), (4, 1, 16, 2), (8, 1, 64, 2),
                                     (2, 2, 8, 2), (3, 2, 12, 3), (4, 2, 32, 3), (8, 2, 64, 3)])
def test_wstar_values(P, V, M, w):
    # SURVEY §8(c) Q4 (scratch-DES facts, re-derived here): W* = 1 / 2 / 3
    assert S.build(cfg_of(P, M, V)).stats[0].w_star == w


@pytest.mark.parametrize("P,V,M", [(4, 1, 16), (4, 2, 32), (8, 1, 64), (8, 2, 64)])
def test_no_added_bubble_encoder(P, V, M):
    # P:202 / P:229: nesting adds no bubble: makespan = T_LLM + per-rank encoder work,
    # which is also the compute-efficient design's time n_u*ef + T_LLM + n_u*eb
    cf, cb, ef, eb = 2, 4, 1, 2
    s = S.build(cfg_of(P, M, V, gen_place="none"))
    mk, _ = simulate(s.ranks, uniform_cost(cf, cb, ef, eb))
    t_llm = (M * V + P - 1) * (cf + cb)
    n_u = M // P
    assert mk == t_llm + n_u * (ef + eb)


def test_generator_program_order_costs_time():
    # per-mb DP-sharded generator run in program order adds time
    # when t_b = 2 t_f (documented reading; motivates the high-priority gen stream)
    s = S.build(cfg_of(8, 64, 1))
    mk, _ = simulate(s.ranks, uniform_cost(4, 8, 2, 4, 3, 6))
    ideal = 71 * 12 + 8 * 6 + 64 * 9
    assert mk > ideal


# --------------------------------------------------------------------------- errors
def test_errors():
    with pytest.raises(S.ScheduleError) as e:
        S.build(cfg_of(4, 63, 1))                  # S:471 remainder
    assert e.value.code == S.E_REMAINDER
    with pytest.raises(S.ScheduleError) as e:
        S.build(cfg_of(4, 32, 2, warmup_units=2))  # S:153 warmup too small (W* = 3)
    assert e.value.code == S.E_WARMUP
    with pytest.raises(S.ScheduleError) as e:
        S.build(S.SchedCfg(2, 4, 2, llm_sched="1f1b"))
    assert e.value.code == S.E_INVALID


# --------------------------------------------------------------------------- A4 comm
@pytest.mark.parametrize("P,V,M", [(2, 1, 4), (4, 1, 16), (4, 2, 32), (4, 2, 64), (8, 1, 64), (8, 2, 64)])
def test_comm_counts_and_conservation(P, V, M):
    s = S.build(cfg_of(P, M, V))
    sends = [(r, o) for r in range(P) for o in s.ranks[r] if o.kind == "Send"]
    recvs = [(r, o) for r in range(P) for o in s.ranks[r] if o.kind == "Recv"]
    cnt = lambda p: sum(1 for _, o in sends if o.payload == p)
    # stage boundaries incl. the chunk wrap P-1 -> 0 (S:251 says M*V*(P-1))
    assert cnt("act") == cnt("grad") == M * (P * V - 1)
    assert cnt("emb") == cnt("embgrad") == M - M // P          # gather / scatter
    assert cnt("genin") == cnt("gengrad") == M * (P - 1)
    # S:264 conservation: every Send has exactly one Recv with equal payload / mb / seq
    sk = sorted((r, o.peer, o.payload, o.seq, o.mb, o.slot) for r, o in sends)
    rk = sorted((o.peer, r, o.payload, o.seq, o.mb, o.slot) for r, o in recvs)
    assert sk == rk
    # S:265 erasing comm ops recovers the compute schedule (order unchanged)
    lists, _ = S.nest(s.cfg, s.llm_base, s.times)
    for r in range(P):
        assert [o for o in s.ranks[r] if o.kind in S.COMPUTE_KINDS] == lists[r]


def test_survey_total_op_counts():
    # SURVEY Appendix A.5 totals (incl. comm): 80, 720, 2208, 5984, 9056
    tot = lambda P, M, V: sum(len(x) for x in S.build(cfg_of(P, M, V)).ranks)
    assert [tot(2, 4, 1), tot(4, 16, 1), tot(4, 32, 2), tot(8, 64, 1), tot(8, 64, 2)] == \
        [80, 720, 2208, 5984, 9056]


def test_paper_setting_send_count_correction():
    # S:251 would give 384 forward sends at (P=4, V=2, M=64); the chunk wrap adds 64
    s = S.build(cfg_of(4, 64, 2))
    assert sum(1 for ops in s.ranks for o in ops if o.kind == "Send" and o.payload == "act") == 448


# --------------------------------------------------------------------------- A5 mutations
def test_mutation_bwd_before_fwd_detected():
    # B0 before F0 on rank 0 -> one violation naming that edge
    s = S.build(cfg_of(2, 4, 1))
    comp = [[o for o in ops if o.kind in S.COMPUTE_KINDS] for ops in s.ranks]
    r0 = comp[0]
    f0 = next(i for i, o in enumerate(r0) if o.kind == "LlmFwd" and o.mb == 0)
    b0 = next(i for i, o in enumerate(r0) if o.kind == "LlmBwd" and o.mb == 0)
    r0.insert(f0, r0.pop(b0))
    assert S.verify_dependencies(s.cfg, comp) != []


def test_mutation_g0_after_f3_detected():
    # moving G_0 after F_3 breaks the order property for unit 0
    s = S.build(cfg_of(4, 64, 2))
    ops = list(s.ranks[0])
    g0 = next(i for i, o in enumerate(ops) if o.kind == "LlmBwd" and o.mb == 3 and o.chunk == 0)
    f3 = next(i for i, o in enumerate(ops) if o.kind == "LlmFwd" and o.mb == 12 and o.chunk == 0)
    g = ops.pop(g0)
    ops.insert(f3, g)
    res = dict(S.order_property(s.cfg, ops))
    assert res[0] is False


def test_mutation_circular_wait_detected():
    # two ranks each waiting on the other before sending -> deadlock
    s = S.build(cfg_of(2, 4, 1))
    ranks = [list(x) for x in s.ranks]
    # rank 0 waits for grad(0) before running F(0) whose output rank 1 needs first
    i_recv = next(i for i, o in enumerate(ranks[0]) if o.kind == "Recv" and o.payload == "grad")
    i_f0 = next(i for i, o in enumerate(ranks[0]) if o.kind == "LlmFwd" and o.mb == 0)
    r = ranks[0].pop(i_recv)
    ranks[0].insert(i_f0, r)
    nid, n, sa, ra, rel = S._index(ranks)
    assert not S._acyclic(n, S._base_edges(ranks, nid, sa, ra))


@pytest.mark.parametrize("P,V,M", [(2, 1, 4), (4, 1, 16), (4, 2, 32), (8, 1, 64)])
def test_rings_are_credit_safe_and_minimal(P, V, M):
    # P:317 deadlock_check with bounded receive slots: all credit edges acyclic, and
    # one slot fewer (without slack) on any channel would deadlock or is the floor 1
    s = S.build(cfg_of(P, M, V, ring_slack=0))
    ranks = s.ranks
    nid, n, sa, ra, rel = S._index(ranks)
    base = S._base_edges(ranks, nid, sa, ra)
    counts = {}
    for r in range(P):
        for o in ranks[r]:
            if o.kind == "Send":
                counts[(r, o.peer, o.payload)] = counts.get((r, o.peer, o.payload), 0) + 1
    allc = []
    for ch, K in s.rings.items():
        allc += S._credit_edges(ch, K, counts[ch], nid, sa, rel)
    assert S._acyclic(n, base + allc)
    for ch, K in s.rings.items():
        if K > 1:
            assert not S._acyclic(n, base + S._credit_edges(ch, K - 1, counts[ch], nid, sa, rel))


def test_serialization_golden():
    # golden file written by scripts/make_golden.py (calls oracle/ only)
    import os
    path = os.path.join(os.path.dirname(__file__), "golden", "sched_P2_M4_V1.tsv")
    with open(path) as f:
        assert S.serialize(S.build(cfg_of(2, 4, 1))) == f.read()


# --------------------------------------------------------------------------- f1 baselines
def test_memory_efficient_baseline_structure():
    # S:204 / P:150-151 (Fig. 3): EncFwd(mb) immediately precedes the entry-stage F(mb, 0);
    # S:205 / P:164: peak live encoder microbatches on rank 0 <= P; S:206 strict chain at P=1
    s = S.build(cfg_of(4, 8, 1, enc_place="entry_stage", gen_place="last_stage"))
    ops0 = [o for o in s.ranks[0] if o.kind in S.COMPUTE_KINDS]
    for i, o in enumerate(ops0):
        if o.kind == "LlmFwd":
            assert ops0[i - 1].kind == "EncFwd" and ops0[i - 1].mb == o.mb
        if o.kind == "LlmBwd":
            assert ops0[i + 1].kind == "EncBwd" and ops0[i + 1].mb == o.mb
    assert s.stats[0].peak_enc_units == 4 and all(st.peak_enc_units == 0 for st in s.stats[1:])
    assert all(o.kind not in ("EncFwd", "EncBwd") for r in range(1, 4) for o in s.ranks[r])
    assert not any(o.payload in ("emb", "embgrad") for ops in s.ranks for o in ops)
    t = S.build(cfg_of(1, 2, 1, enc_place="entry_stage", gen_place="last_stage"))
    assert [o.kind for o in t.ranks[0]] == ["EncFwd", "LlmFwd", "GenFwd", "GenBwd", "LlmBwd", "EncBwd",
                                            "EncFwd", "LlmFwd", "GenFwd", "GenBwd", "LlmBwd", "EncBwd"]


@pytest.mark.parametrize("P,M", [(4, 16), (4, 64), (2, 8)])
def test_compute_efficient_baseline_memory(P, M):
    # S:195-196 / P:132: all encoder forwards first -> (M/P) live units per rank,
    # i.e. memory that grows with M, while BigMac's window stays at W*
    ce = S.build(cfg_of(P, M, 1, warmup_units=M // P))
    ops0 = ce.ranks[0]
    first_llm = next(i for i, o in enumerate(ops0) if o.kind == "LlmFwd")
    assert sum(1 for o in ops0[:first_llm] if o.kind == "EncFwd") == M // P
    assert all(st.peak_enc_units == M // P for st in ce.stats)
    bm = S.build(cfg_of(P, M, 1))
    assert all(st.peak_enc_units == bm.stats[0].w_star for st in bm.stats)


def test_bigmac_vs_baselines_des():
    # P:229 / S:305: BigMac matches the compute-efficient time; S:315 / S:552: with
    # heterogeneous encoder costs the memory-efficient pipeline is strictly slower
    P, M = 4, 16
    enc_cost = [1 if m % 2 else 3 for m in range(M)]

    def cost(r, op):
        if op.kind in ("EncFwd", "EncBwd"):
            return enc_cost[op.mb] * (1 if op.kind == "EncFwd" else 2)
        return {"LlmFwd": 2, "LlmBwd": 4, "GenFwd": 0, "GenBwd": 0}[op.kind]
    bigmac = simulate(S.build(cfg_of(P, M, 1, gen_place="none")).ranks, cost)[0]
    ce = simulate(S.build(cfg_of(P, M, 1, gen_place="none", warmup_units=M // P)).ranks, cost)[0]
    me = simulate(S.build(cfg_of(P, M, 1, enc_place="entry_stage", gen_place="none")).ranks, cost)[0]
    assert me > bigmac
    # per-rank encoder work differs across ranks (data heterogeneity), so both DP designs
    # pay the slowest rank's encoder time per unit; BigMac never exceeds compute-efficient
    assert bigmac <= ce
