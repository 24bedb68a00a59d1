"""C++ schedule builder (through the C ABI) vs the oracle: byte-identical
serialization, identical statistics and ring sizes, identical error codes.
CPU-only (no GPU needed to build schedules)."""
import pytest

from oracle import schedule as S

L = pytest.importorskip("paper_2605_25451_b200._lib")
from paper_2605_25451_b200 import schedule as BS  # noqa: E402

GRID = [(P, M, V) for P in (1, 2, 3, 4, 8) for V in (1, 2, 4) for M in (P, 2 * P, 8 * P)]
GRID += [(4, 64, 2), (8, 64, 1), (8, 64, 2), (4, 16, 1), (4, 32, 2), (2, 4, 1)]


def both(P, M, V, **kw):
    sched = "1f1b" if V == 1 else "interleaved"
    o = S.build(S.SchedCfg(P, M, V, llm_sched=sched, **kw))
    c = BS.build(P, M, V, **kw)
    return o, c


@pytest.mark.parametrize("P,M,V", GRID)
@pytest.mark.parametrize("kw", [{}, {"cost_fwd": 1, "cost_bwd": 1}, {"gen_place": "last_stage"},
                                {"gen_place": "none", "ring_slack": 0}, {"warmup_units": 3},
                                {"enc_place": "entry_stage", "gen_place": "last_stage"},
                                {"enc_place": "entry_stage", "gen_place": "dp_shard"},
                                {"enc_exclude": 1}, {"enc_exclude": 4}, {"enc_exclude": 6, "gen_place": "last_stage"}])
def test_serialization_identical(P, M, V, kw):
    try:
        o = S.build(S.SchedCfg(P, M, V, llm_sched="1f1b" if V == 1 else "interleaved", **kw))
    except S.ScheduleError as e:
        with pytest.raises(L.BigMacError) as ce:
            BS.build(P, M, V, **kw)
        assert ce.value.code == e.code
        return
    c = BS.build(P, M, V, **kw)
    assert c.serialize() == S.serialize(o)
    for r in range(P):
        st, so = c.stats(r), o.stats[r]
        assert (st.w_star, st.warmup_units, st.peak_enc_units, st.peak_gen_shards, st.peak_llm_inflight,
                st.n_ops, st.llm_idle_cost_units, st.makespan_cost_units) == \
            (so.w_star, so.warmup_units, so.peak_enc_units, so.peak_gen_shards, so.peak_llm_inflight,
             so.n_ops, so.llm_idle_cost_units, so.makespan_cost_units)
        assert list(st.ring_slots) == [so.ring_slots[p] for p in S.PAYLOADS]
    for (src, dst, pay), K in o.rings.items():
        assert c.ring(src, dst, S.PAYLOADS.index(pay))[0] == K


@pytest.mark.parametrize("args,code", [((4, 63, 1), 2), ((4, 32, 2, 2), 3)])
def test_error_codes(args, code):
    P, M, V = args[:3]
    kw = {"warmup_units": args[3]} if len(args) > 3 else {}
    with pytest.raises(L.BigMacError) as e:
        BS.build(P, M, V, **kw)
    assert e.value.code == code


def test_invalid_v_for_1f1b():
    with pytest.raises(L.BigMacError) as e:
        BS.build(2, 4, 2, llm_sched="1f1b")
    assert e.value.code == 1


def test_golden_file():
    import os
    path = os.path.join(os.path.dirname(__file__), "golden", "sched_P4_M8_V2.tsv")
    with open(path) as f:
        assert BS.build(4, 8, 2).serialize() == f.read()


ZB_GRID = [(P, M) for P in (1, 2, 3, 4, 8) for M in (P, 2 * P, 8 * P)] + [(4, 64), (8, 64), (8, 256)]


@pytest.mark.parametrize("P,M", ZB_GRID)
@pytest.mark.parametrize("kw", [{}, {"cost_fwd": 2, "cost_bwd": 4, "cost_wgrad": 1}, {"cost_fwd": 1, "cost_bwd": 3},
                                {"gen_place": "last_stage"}, {"gen_place": "none", "ring_slack": 0},
                                {"enc_place": "entry_stage", "gen_place": "last_stage"}, {"enc_exclude": 1}])
def test_zb_h1_serialization_identical(P, M, kw):
    """ZB-H1 (reading R23): the C++ builder's B/W split lists equal the oracle's."""
    try:
        o = S.build(S.SchedCfg(P, M, 1, llm_sched="zb_h1", **kw))
    except S.ScheduleError as e:
        with pytest.raises(L.BigMacError) as ce:
            BS.build(P, M, 1, llm_sched="zb_h1", **kw)
        assert ce.value.code == e.code
        return
    c = BS.build(P, M, 1, llm_sched="zb_h1", **kw)
    assert c.serialize() == S.serialize(o)
    for r in range(P):
        st, so = c.stats(r), o.stats[r]
        assert (st.w_star, st.peak_enc_units, st.peak_gen_shards, st.peak_llm_inflight, st.n_ops,
                st.llm_idle_cost_units, st.makespan_cost_units) == \
            (so.w_star, so.peak_enc_units, so.peak_gen_shards, so.peak_llm_inflight, so.n_ops,
             so.llm_idle_cost_units, so.makespan_cost_units)


@pytest.mark.parametrize("kw", [{"cost_bwd": 1}, {"cost_bwd": 2, "cost_wgrad": 2}, {"cost_wgrad": -1}])
def test_zb_h1_invalid_costs(kw):
    with pytest.raises(S.ScheduleError) as e:
        S.build(S.SchedCfg(4, 8, 1, llm_sched="zb_h1", **kw))
    with pytest.raises(L.BigMacError) as ce:
        BS.build(4, 8, 1, llm_sched="zb_h1", **kw)
    assert ce.value.code == e.value.code == 1


def test_zb_h1_requires_v1():
    with pytest.raises(L.BigMacError) as e:
        BS.build(2, 4, 2, llm_sched="zb_h1")
    assert e.value.code == 1


CP_GRID = [(4, 16, 1, 2, 1), (4, 32, 1, 2, 2), (2, 8, 1, 2, 1), (2, 8, 1, 4, 2), (4, 32, 2, 2, 1),
           (2, 12, 1, 3, 1), (3, 12, 1, 2, 1), (2, 16, 1, 4, 1), (8, 64, 1, 2, 1), (4, 12, 1, 2, 1), (2, 8, 1, 1, 2)]


@pytest.mark.parametrize("P,M,V,lcp,ecp", CP_GRID)
@pytest.mark.parametrize("kw", [{"gen_place": "last_stage"}, {"gen_place": "none"}, {"enc_place": "none", "gen_place": "none"},
                                {"gen_place": "last_stage", "llm_sched": "zb_h1"}, {"gen_place": "last_stage", "warmup_units": 3},
                                {"gen_place": "dp_shard"}])
def test_cp_serialization_identical(P, M, V, lcp, ecp, kw):
    """Decoupled CP (reading R25): the C++ builder's P llm_cp-rank lists equal the oracle's."""
    kw = dict(kw)
    sched = kw.pop("llm_sched", "1f1b" if V == 1 else "interleaved")
    if sched == "zb_h1" and V != 1:
        pytest.skip("ZB-H1 needs V = 1")
    try:
        o = S.build(S.SchedCfg(P, M, V, llm_sched=sched, llm_cp=lcp, enc_cp=ecp, **kw))
    except S.ScheduleError as e:
        with pytest.raises(L.BigMacError) as ce:
            BS.build(P, M, V, llm_sched=sched, llm_cp=lcp, enc_cp=ecp, **kw)
        assert ce.value.code == e.code
        return
    c = BS.build(P, M, V, llm_sched=sched, llm_cp=lcp, enc_cp=ecp, **kw)
    assert c.serialize() == S.serialize(o)
    for k in range(P * lcp):
        st, so = c.stats(k), o.stats[k]
        assert (st.w_star, st.warmup_units, st.peak_enc_units, st.peak_gen_shards, st.peak_llm_inflight, st.n_ops,
                st.llm_idle_cost_units, st.makespan_cost_units) == \
            (so.w_star, so.warmup_units, so.peak_enc_units, so.peak_gen_shards, so.peak_llm_inflight, so.n_ops,
             so.llm_idle_cost_units, so.makespan_cost_units)
