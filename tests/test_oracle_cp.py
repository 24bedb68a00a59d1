"""Pins for the decoupled context-parallel schedule (reading R25).

The oracle's build_cp nests the encoder into the LLM schedule of P * llm_cp ranks
(rank c P + r = LLM CP index c, stage r) with encoder units of P llm_cp / enc_cp
microbatches and the encoder-to-LLM CP-conversion all-to-all expanded into P2P
messages.  These tests check it against what the paper fixes, with machinery
written here (independent DES, token-game executor, textbook 1F1B lists):

* with llm_cp = enc_cp = 1 it is the paper's base nesting (byte-identical to build);
* the unit is P llm_cp / enc_cp microbatches (LLM CP 2, encoder CP 1, P = 4
  -> eight), every microbatch encoded once by each rank of its encoder CP group;
* every rank runs its stage's LLM list unchanged ("preserving the original LLM
  pipeline order");
* CP-conversion message counts (every encoder-group rank to every stage-0 CP rank
  and back), send/recv conservation;
* dependency safety and no added bubble in an independent DES with the all-to-all
  dependencies; the executor token game completes with the oracle's rings;
* encoder activations stay within W units per rank.
"""

import pytest

from oracle import schedule as S

from test_oracle_pins_r2 import token_game  # noqa: E402


def cfg_of(P, M, V=1, **kw):
    return S.SchedCfg(P, M, V, llm_sched="1f1b" if V == 1 else "interleaved", **kw)


@pytest.mark.parametrize("P,M,V", [(1, 3, 1), (2, 4, 1), (3, 6, 1), (4, 16, 1), (4, 8, 2), (8, 64, 1), (4, 32, 2)])
@pytest.mark.parametrize("kw", [{"gen_place": "last_stage"}, {"gen_place": "none"},
                                {"enc_place": "none", "gen_place": "none"},
                                {"gen_place": "last_stage", "warmup_units": 3}])
def test_cp1_is_the_base_nesting(P, M, V, kw):
    c = cfg_of(P, M, V, **kw)
    assert S.serialize(S.build_cp(c)) == S.serialize(S.build(c))


CP_GRID = [(4, 16, 1, 2, 1), (4, 32, 1, 2, 2), (2, 8, 1, 2, 1), (2, 8, 1, 4, 2), (4, 32, 2, 2, 1),
           (2, 12, 1, 3, 1), (3, 12, 1, 2, 1), (2, 16, 1, 4, 1), (8, 64, 1, 2, 1)]


@pytest.mark.parametrize("P,M,V,lcp,ecp", CP_GRID)
@pytest.mark.parametrize("gen", ["last_stage", "none"])
def test_cp_unit_and_encoder_coverage(P, M, V, lcp, ecp, gen):
    s = S.build(cfg_of(P, M, V, llm_cp=lcp, enc_cp=ecp, gen_place=gen))
    R, U = P * lcp, P * lcp // ecp
    assert len(s.ranks) == R
    for u in range(M // U):
        # each unit covers U consecutive microbatches, each encoded by enc_cp ranks
        owners = {}
        for k in range(R):
            for o in s.ranks[k]:
                if o.kind == "EncFwd" and o.unit == u:
                    owners.setdefault(o.mb, []).append(k)
        assert sorted(owners) == list(range(u * U, u * U + U))
        assert all(len(v) == ecp for v in owners.values())
        assert sorted(k for v in owners.values() for k in v) == list(range(R))   # one per rank
    for k in range(R):
        ops = [o for o in s.ranks[k] if o.kind in ("EncFwd", "EncBwd")]
        assert [o.mb for o in ops if o.kind == "EncFwd"] == [o.mb for o in ops if o.kind == "EncBwd"]


def test_paper_example_eight_microbatch_unit():
    # "LLM CP size two and encoder CP size one yield an eight micro-batch encoder unit"
    s = S.build(cfg_of(4, 16, 1, llm_cp=2, enc_cp=1, gen_place="last_stage"))
    unit0 = sorted(o.mb for ops in s.ranks for o in ops if o.kind == "EncFwd" and o.unit == 0)
    assert unit0 == list(range(8))


def _textbook_1f1b(P, M, r):
    w = min(P - r - 1, M)
    out = [("F", m, 0) for m in range(w)]
    for i in range(M - w):
        out += [("F", w + i, 0), ("B", i, 0)]
    return out + [("B", i, 0) for i in range(M - w, M)]


@pytest.mark.parametrize("P,M,V,lcp,ecp", CP_GRID)
def test_cp_llm_order_and_conversion_messages(P, M, V, lcp, ecp):
    s = S.build(cfg_of(P, M, V, llm_cp=lcp, enc_cp=ecp, gen_place="last_stage"))
    R, U = P * lcp, P * lcp // ecp
    name = {"LlmFwd": "F", "LlmBwd": "B", "LlmW": "W"}
    for k in range(R):
        seq = [(name[o.kind], o.mb, o.chunk) for o in s.ranks[k] if o.kind in name]
        if V == 1:
            assert seq == _textbook_1f1b(P, M, k % P)
        else:
            assert seq == [tuple(x) for x in S.llm_base_schedule(P, M, V)[k % P]]
    # the CP-conversion all-to-all: every encoder-group rank -> every stage-0 CP rank (and back)
    stage0 = [c * P for c in range(lcp)]
    want = sum(1 for m in range(M) for q in range((m % U) * ecp, (m % U + 1) * ecp) for z in stage0 if q != z)
    sends = [o for ops in s.ranks for o in ops if o.kind == "Send"]
    recvs = [o for ops in s.ranks for o in ops if o.kind == "Recv"]
    assert sum(o.payload == "emb" for o in sends) == want == sum(o.payload == "emb" for o in recvs)
    assert sum(o.payload == "embgrad" for o in sends) == want == sum(o.payload == "embgrad" for o in recvs)
    # act / grad stay inside a CP index: M (PV - 1) messages per direction per CP group
    assert sum(o.payload == "act" for o in sends) == lcp * M * (P * V - 1)
    for k, ops in enumerate(s.ranks):
        for o in ops:
            if o.payload in ("act", "grad"):
                assert o.peer // P == k // P


def _des(P, lcp, ecp, lists, cost):
    """Independent DES: program order per rank, data deps incl. the CP all-to-all."""
    U = P * lcp // ecp
    grp = lambda m: range((m % U) * ecp, (m % U + 1) * ecp)   # noqa: E731
    stage0 = [c * P for c in range(lcp)]
    end, ptr, clock = {}, [0] * len(lists), [0] * len(lists)
    n, fired = sum(len(x) for x in lists), 0
    while fired < n:
        moved = False
        for k, ops in enumerate(lists):
            c, r = divmod(k, P)
            while ptr[k] < len(ops):
                o = ops[ptr[k]]
                if o.kind == "LlmFwd":
                    deps = [("LlmFwd", o.mb, c * P + r - 1)] if r else [("EncFwd", o.mb, q) for q in grp(o.mb)]
                elif o.kind == "LlmBwd":
                    deps = [("LlmFwd", o.mb, k)] + ([("LlmBwd", o.mb, k + 1)] if r < P - 1 else [])
                    if r == P - 1 and any(x.kind == "GenBwd" for x in ops):
                        deps.append(("GenBwd", o.mb, k))
                elif o.kind == "EncBwd":
                    deps = [("EncFwd", o.mb, k)] + [("LlmBwd", o.mb, z) for z in stage0]
                elif o.kind == "GenFwd":
                    deps = [("LlmFwd", o.mb, k)]
                elif o.kind == "GenBwd":
                    deps = [("GenFwd", o.mb, k)]
                else:
                    deps = []
                if any(d not in end for d in deps):
                    break
                end[(o.kind, o.mb, k)] = clock[k] = max([clock[k]] + [end[d] for d in deps]) + cost[o.kind]
                ptr[k] += 1
                fired += 1
                moved = True
        if not moved:
            return None
    return max(clock)


@pytest.mark.parametrize("P,M,lcp,ecp", [(4, 16, 2, 1), (2, 8, 2, 1), (2, 8, 4, 2), (4, 32, 2, 2), (3, 12, 2, 1),
                                        (2, 16, 4, 1), (8, 64, 2, 1)])
@pytest.mark.parametrize("ef,eb", [(1, 1), (1, 2)])
def test_cp_no_added_bubble(P, M, lcp, ecp, ef, eb):
    """Nested CP schedule: dependency-safe, and the makespan is the LLM's plus one
    encoder forward and backward per unit (every rank encodes one microbatch shard per
    unit) -- the compute-efficient time at unit costs."""
    s = S.build(cfg_of(P, M, 1, llm_cp=lcp, enc_cp=ecp, gen_place="none", cost_fwd=1, cost_bwd=2))
    U = P * lcp // ecp
    lists = [[o for o in ops if o.kind in S.COMPUTE_KINDS] for ops in s.ranks]
    mk = _des(P, lcp, ecp, lists, {"LlmFwd": 1, "LlmBwd": 2, "EncFwd": ef, "EncBwd": eb})
    assert mk is not None
    t_llm = (M + P - 1) * 3
    assert mk == t_llm + (M // U) * (ef + eb)


@pytest.mark.parametrize("P,M,V,lcp,ecp", CP_GRID)
def test_cp_rings_deadlock_free_and_memory(P, M, V, lcp, ecp):
    s = S.build(cfg_of(P, M, V, llm_cp=lcp, enc_cp=ecp, gen_place="last_stage"))
    assert token_game(s.ranks, s.rings)
    for st in s.stats:
        assert st.peak_enc_units <= st.warmup_units
        assert st.peak_gen_shards <= 1


def test_cp_errors():
    with pytest.raises(S.ScheduleError) as e:           # M not a multiple of the 8-microbatch unit
        S.build(cfg_of(4, 12, 1, llm_cp=2, gen_place="none"))
    assert e.value.code == S.E_REMAINDER
    for kw in ({"llm_cp": 2, "enc_cp": 3}, {"llm_cp": 0}, {"llm_cp": 2}, {"llm_cp": 1, "enc_cp": 2},
               {"llm_cp": 2, "enc_place": "entry_stage", "gen_place": "none"}):
        with pytest.raises(S.ScheduleError) as e:        # bad degrees; DP-sharded generator with CP
            S.build(cfg_of(4, 16, 1, **kw))
        assert e.value.code == S.E_INVALID


@pytest.mark.parametrize("P,M,V,lcp,ecp,edge,zb", [(2, 8, 1, 2, 1, False, False), (2, 8, 1, 2, 2, False, False),
                                                   (4, 16, 1, 2, 1, False, False), (2, 8, 1, 4, 2, False, False),
                                                   (2, 8, 2, 2, 1, False, False), (2, 16, 1, 4, 1, False, False),
                                                   (2, 8, 1, 2, 2, True, False), (4, 16, 1, 2, 1, True, False),
                                                   (2, 8, 1, 2, 1, False, True), (4, 16, 1, 2, 2, True, True)])
def test_cp_interpreter_equals_sequential(P, M, V, lcp, ecp, edge, zb):
    """The fp64 interpreter executes the CP schedule with sequence-sharded LLM ranks,
    row-sharded encoder CP groups and the CP-conversion messages carrying the row
    intersections; loss and every gradient equal the sequential reference,
    including the degenerate batches (no modality rows, no text rows, overlapping
    generator rows, fewer generator rows than ranks)."""
    import numpy as np
    from synth import edge_counts, edge_shape, get_config, make_batch, make_weights
    from oracle import interp
    from oracle import model as om
    cfg = get_config("C1", P=P, M=M, V=V)
    if V > 1:
        cfg = cfg.replace(llm_sched="interleaved")
    if edge:
        cfg = edge_shape(cfg)
        n_mod, n_gen = edge_counts(cfg, M)
        W, B = make_weights(cfg), make_batch(cfg, n_mod=n_mod, n_gen=n_gen)
    else:
        W, B = make_weights(cfg), make_batch(cfg)
    loss, per, G = om.step_fp64(cfg, W, B)
    kw = {"llm_sched": "zb_h1"} if zb else {}
    s = S.build(S.SchedCfg(P, M, V, llm_sched=kw.get("llm_sched", "1f1b" if V == 1 else "interleaved"),
                           llm_cp=lcp, enc_cp=ecp, gen_place="last_stage"))
    loss2, per2, G2 = interp.run_cp(s, cfg, W, B)
    assert abs(loss2 - loss) <= 1e-12 * abs(loss)
    assert np.allclose(per2, per, rtol=1e-12, atol=1e-15)
    for k in G:
        assert np.linalg.norm(G2[k] - G[k]) <= 1e-12 * max(np.linalg.norm(G[k]), 1e-30), k
