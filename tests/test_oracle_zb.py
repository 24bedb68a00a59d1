"""Pins for the zero-bubble base schedule (ZB-H1, reading R23).

P:552-556 names zero-bubble pipeline parallelism (Qi et al.) as the LLM
schedule class BigMac should extend to.  The oracle builds ZB-H1 by the rule in
oracle/schedule.zb_h1_schedule; these tests check its output against what the
zero-bubble construction fixes, with machinery written here (an independent
DES, textbook 1F1B lists), never with the oracle's own des_llm:

* per-rank idle time (P-1)(T_F + T_B - T_W) when T_W <= min(T_F, T_B)
  (ZB-H1's bubble, a third of 1F1B's (P-1)(T_F + T_B + T_W) at equal costs);
* every rank keeps the 1F1B order of its F and B ops;
* no rank holds more than P microbatches between F and W (1F1B's peak, rank 0);
* at equal costs rank r runs W(m) right after B(m + r) in the steady phase
  (the ZB-H1 figure: stage r defers r weight-gradient ops);
* nesting the encoder / generator into ZB-H1 keeps the LLM order, adds no
  bubble (makespan = T_LLM + encoder work) and stays dependency-safe;
* the fp64 interpreter with B = input gradient and W = the deferred dY^T X
  products reaches the sequential gradients.
"""
import numpy as np
import pytest

from oracle import schedule as S

GRID = [(2, 4), (2, 8), (3, 6), (4, 4), (4, 8), (4, 16), (8, 16), (8, 64)]
COSTS = [(1, 1, 1), (2, 2, 1), (2, 3, 2), (3, 2, 2), (1, 2, 1), (2, 1, 1), (3, 3, 2), (4, 3, 3), (5, 4, 2)]


def textbook_1f1b(P, M, r):
    w = min(P - r - 1, M)
    out = [("F", m) for m in range(w)]
    for i in range(M - w):
        out += [("F", w + i), ("B", i)]
    return out + [("B", i) for i in range(M - w, M)]


def indep_des(P, lists, cf, cb, cw):
    """F(m, r) after F(m, r-1); B(m, r) after B(m, r+1) and F(m, r); W(m, r) after
    B(m, r); each rank in list order.  Returns (makespan, busy per rank) or None."""
    end, ptr, clock = {}, [0] * P, [0] * P
    cost = {"F": cf, "B": cb, "W": cw}
    n, fired = sum(len(x) for x in lists), 0
    while fired < n:
        moved = False
        for r in range(P):
            while ptr[r] < len(lists[r]):
                k, m = lists[r][ptr[r]][:2]
                deps = {"F": [(r - 1, "F", m)] if r else [],
                        "B": [(r, "F", m)] + ([(r + 1, "B", m)] if r < P - 1 else []),
                        "W": [(r, "B", m)]}[k]
                if any(d not in end for d in deps):
                    break
                t0 = max([clock[r]] + [end[d] for d in deps])
                end[(r, k, m)] = clock[r] = t0 + cost[k]
                ptr[r] += 1
                fired += 1
                moved = True
        if not moved:
            return None
    return max(clock)


def zb_cfg(P, M, cf, cb, cw, **kw):
    return S.SchedCfg(P, M, 1, llm_sched="zb_h1", cost_fwd=cf, cost_bwd=cb + cw, cost_wgrad=cw, **kw)


@pytest.mark.parametrize("P,M", GRID)
@pytest.mark.parametrize("cf,cb,cw", COSTS)
def test_zb_h1_bubble_closed_form(P, M, cf, cb, cw):
    s = S.build(zb_cfg(P, M, cf, cb, cw, enc_place="none", gen_place="none"))
    lists = [[(k, m) for k, m, _ in s.llm_base[r]] for r in range(P)]
    mk = indep_des(P, lists, cf, cb, cw)
    assert mk is not None
    idle = (P - 1) * (cf + cb - cw)            # ZB-H1 (Qi et al.), valid for cw <= min(cf, cb)
    assert mk == M * (cf + cb + cw) + idle
    for st in s.stats:
        assert st.makespan_cost_units == mk
        assert st.llm_idle_cost_units == idle


@pytest.mark.parametrize("P,M", GRID)
def test_zb_h1_third_of_1f1b_bubble(P, M):
    zb = S.build(zb_cfg(P, M, 1, 1, 1, enc_place="none", gen_place="none"))
    ref = S.build(S.SchedCfg(P, M, 1, cost_fwd=1, cost_bwd=2, enc_place="none", gen_place="none"))
    assert ref.stats[0].llm_idle_cost_units == 3 * (P - 1)
    assert 3 * zb.stats[0].llm_idle_cost_units == ref.stats[0].llm_idle_cost_units


@pytest.mark.parametrize("P,M", GRID)
@pytest.mark.parametrize("cf,cb,cw", COSTS)
def test_zb_h1_keeps_1f1b_order_and_memory(P, M, cf, cb, cw):
    s = S.build(zb_cfg(P, M, cf, cb, cw))
    for r in range(P):
        fb = [(k, m) for k, m, _ in s.llm_base[r] if k != "W"]
        assert fb == textbook_1f1b(P, M, r)
        # every B(m) has exactly one W(m) after it
        ws = [m for k, m, _ in s.llm_base[r] if k == "W"]
        assert sorted(ws) == list(range(M))
        pos = {(k, m): i for i, (k, m, _) in enumerate(s.llm_base[r])}
        assert all(pos[("B", m)] < pos[("W", m)] for m in range(M))
        held = peak = 0
        for k, m, _ in s.llm_base[r]:
            held += {"F": 1, "B": 0, "W": -1}[k]
            peak = max(peak, held)
        assert peak <= P and s.stats[r].peak_llm_inflight == peak
    assert max(st.peak_llm_inflight for st in s.stats) == min(P, M)   # 1F1B's rank-0 peak


@pytest.mark.parametrize("P,M", [(4, 16), (8, 64), (3, 9), (2, 8)])
def test_zb_h1_figure_structure(P, M):
    s = S.build(zb_cfg(P, M, 1, 1, 1))
    for r in range(P):
        ops = [(k, m) for k, m, _ in s.llm_base[r]]
        for m in range(M - r):
            i = ops.index(("B", m + r))
            if m + r < M - (P - r - 1):        # steady phase: an F follows
                assert ops[i + 1] == ("W", m), (r, m, ops)


@pytest.mark.parametrize("P,M,ef,eb", [(2, 4, 1, 1), (4, 8, 1, 2), (4, 16, 2, 3), (3, 6, 1, 1)])
def test_zb_h1_nesting_adds_no_bubble(P, M, ef, eb):
    """Encoder nested into ZB-H1: LLM order unchanged and, in an
    independent DES where EncFwd(u) / EncBwd(u) cost ef / eb on every rank, the
    makespan is T_LLM + n_u (ef + eb) -- the compute-efficient time."""
    cf, cb, cw = 1, 1, 1
    s = S.build(zb_cfg(P, M, cf, cb, cw, gen_place="none"))
    n_u = M // P
    lists = []
    for r in range(P):
        ops = [o for o in s.ranks[r] if o.kind in S.COMPUTE_KINDS]
        assert [(k, m) for k, m, _ in s.llm_base[r]] == \
            [({"LlmFwd": "F", "LlmBwd": "B", "LlmW": "W"}[o.kind], o.mb) for o in ops if o.kind.startswith("Llm")]
        lists.append(ops)
    end, ptr, clock = {}, [0] * P, [0] * P
    cost = {"LlmFwd": cf, "LlmBwd": cb, "LlmW": cw, "EncFwd": ef, "EncBwd": eb}
    n, fired = sum(len(x) for x in lists), 0
    while fired < n:
        moved = False
        for r in range(P):
            while ptr[r] < len(lists[r]):
                o = lists[r][ptr[r]]
                key = (o.kind, o.mb, r)
                if o.kind == "LlmFwd":
                    deps = [("LlmFwd", o.mb, r - 1)] if r else [("EncFwd", o.mb, o.mb % P)]
                elif o.kind == "LlmBwd":
                    deps = [("LlmFwd", o.mb, r)] + ([("LlmBwd", o.mb, r + 1)] if r < P - 1 else [])
                elif o.kind == "LlmW":
                    deps = [("LlmBwd", o.mb, r)]
                elif o.kind == "EncBwd":
                    deps = [("LlmBwd", o.mb, 0), ("EncFwd", o.mb, r)]
                else:
                    deps = []
                if any(d not in end for d in deps):
                    break
                end[key] = clock[r] = max([clock[r]] + [end[d] for d in deps]) + cost[o.kind]
                ptr[r] += 1
                fired += 1
                moved = True
        assert moved, "nested ZB-H1 schedule deadlocks"
    t_llm = M * (cf + cb + cw) + (P - 1) * (cf + cb - cw)
    assert max(clock) == t_llm + n_u * (ef + eb)


@pytest.mark.parametrize("P,M,L,kw", [(2, 4, 4, {}), (4, 16, 4, {}), (4, 8, 4, {"gen_place": "last_stage"}),
                                      (2, 4, 2, {"enc_place": "entry_stage", "gen_place": "last_stage"}),
                                      (1, 3, 2, {}), (4, 8, 8, {"cost_fwd": 2, "cost_bwd": 4, "cost_wgrad": 1})])
def test_zb_h1_interpreter_equals_sequential(P, M, L, kw):
    from synth import get_config, make_batch, make_weights
    from oracle import interp
    from oracle import model as om
    cfg = get_config("C1", P=P, M=M).replace(L=L)
    W, B = make_weights(cfg), make_batch(cfg)
    loss, per, G = om.step_fp64(cfg, W, B)
    sched = S.build(S.SchedCfg(P, M, 1, llm_sched="zb_h1", **kw))
    loss2, per2, G2, _ = interp.run(sched, cfg, W, B)
    assert abs(loss2 - loss) <= 1e-12 * abs(loss)
    assert per2 == per or np.allclose(per2, per, rtol=1e-13, atol=0)
    for k in G:
        assert np.linalg.norm(G2[k] - G[k]) <= 1e-12 * max(np.linalg.norm(G[k]), 1e-30), k


def test_zb_h1_rejects_bad_costs():
    for kw in ({"cost_bwd": 1}, {"cost_bwd": 2, "cost_wgrad": 2}, {"cost_wgrad": -1}):
        with pytest.raises(S.ScheduleError) as e:
            S.build(S.SchedCfg(4, 8, 1, llm_sched="zb_h1", **kw))
        assert e.value.code == S.E_INVALID
    with pytest.raises(S.ScheduleError):
        S.build(S.SchedCfg(4, 8, 2, llm_sched="zb_h1"))
