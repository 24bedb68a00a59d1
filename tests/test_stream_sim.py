"""Executor stream semantics are deadlock-free (CPU).

tests/tools/stream_sim.py replays bm_step's enqueue logic (compute, generator,
encoder and per-peer comm streams; data/credit flag waits; producer, Hn,
copy-done, generator-done, encoder-output and embedding-gradient events; the step-end allreduce barrier) as FIFO streams on the
schedule the oracle builds, and runs them to completion.  A stuck stream means
the executor adds a dependency cycle that the schedule's own acyclicity check
(oracle/schedule.py size_rings) does not see."""
import os
import sys

import pytest

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "tools"))
from oracle import schedule as S  # noqa: E402
from stream_sim import simulate  # noqa: E402

CASES = [(P, M, V) for P in (1, 2, 3, 4) for M in (P, 2 * P, 4 * P) for V in (1, 2)] + [(8, 16, 1), (8, 16, 2)]
PLACEMENTS = [{}, {"gen_place": "last_stage"}, {"enc_place": "entry_stage", "gen_place": "last_stage"},
              {"gen_place": "none"}]


@pytest.mark.parametrize("P,M,V", CASES)
@pytest.mark.parametrize("kw", PLACEMENTS + [{"warmup": "M/P"}, {"warmup_units": 2}, {"warmup_units": 3}])
def test_no_executor_deadlock(P, M, V, kw):
    kw = dict(kw)
    if kw.pop("warmup", None):
        kw["warmup_units"] = M // P           # compute-efficient baseline
    try:
        sched = S.build(S.SchedCfg(P, M, V, llm_sched="1f1b" if V == 1 else "interleaved", **kw))
    except S.ScheduleError:
        pytest.skip("configuration rejected by the builder")
    stuck = simulate(sched, steps=2)
    assert not stuck, stuck
    # encoder stream forced on at any P (BM_ENC_STREAM=1); the default has it at P = 1
    stuck = simulate(sched, steps=2, use_enc_stream=True)
    assert not stuck, stuck
