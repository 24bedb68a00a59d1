"""Host-side logic of bench.py (no GPU): the workload each N runs, the layer
partition rules, the algorithmic FLOP count against SURVEY.md §8(d)'s table,
and the reference arm's JSON line (the oracle timed on a tiny sample)."""
import argparse
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def ns(**kw):
    d = dict(config="C2", microbatches=0, stages=0, last_stage_layers=-1, stage_layers="")
    d.update(kw)
    return argparse.Namespace(**d)


@pytest.mark.parametrize("N,P,D,M", [(1, 1, 1, 16), (2, 2, 1, 32), (4, 4, 1, 64), (8, 4, 2, 64)])
def test_workload_ladder(N, P, D, M):
    # SURVEY §8(d) GPU ladder: P = G up to 4 stages, then pipeline replicas; 16 microbatches per GPU
    cfg, p, d = bench.workload(ns(), N)
    assert (p, d, cfg.M, cfg.V) == (P, D, M, 1)
    assert cfg.M * d == 16 * N
    cfg3, p3, _ = bench.workload(ns(config="C3"), 4)
    assert (cfg3.V, p3, cfg3.M % p3) == (2, 4, 0)


def test_layer_partition_rules():
    a = ns()
    for N, expect in [(2, 7), (4, 3), (8, 3)]:
        cfg, P, _ = bench.workload(a, N)
        assert bench.last_stage_layers(a, cfg, P) == expect
    cfg, P, _ = bench.workload(a, 4)
    split = bench.stage_split(a, cfg, P)
    assert sum(split) == cfg.L and len(split) == P
    assert bench.stage_split(ns(stage_layers="5,4,4,3"), cfg, P) == [5, 4, 4, 3]
    assert bench.last_stage_layers(a, *bench.workload(a, 1)[:2]) == 0


def test_step_flops_matches_survey_table():
    # FLOP per microbatch at the mean modality / generation rows:
    # C2 21.3 TF (LLM 93.0 %), C4 220.4 TF (LLM 96.5 %)
    from synth import get_config
    for name, n_mean, total, llm_share in [("C2", 554, 21.3e12, 0.930), ("C4", 1385, 220.4e12, 0.965)]:
        cfg = get_config(name, P=1, M=1)
        f = bench.step_flops(cfg, [n_mean], [n_mean])
        llm = 6.0 * cfg.S * 3 * cfg.d * cfg.f * cfg.L
        assert abs(f - total) / total < 0.01, (name, f)
        assert abs(llm / f - llm_share) < 0.005, (name, llm / f)


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "0", "--ref-seq-div", "32"], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "oracle"
    assert line["config"]["workload"].startswith("C2")


def test_bubble_from_trace_closed_form():
    # compute-stream busy [0,2] u [1,3] u [5,6] over a step ending at 8 -> idle 4/8;
    # receives, other streams and the tail do not count as busy
    recs = [{"t0": 0.0, "t1": 2.0, "stream": 0, "kind": "LlmFwd"}, {"t0": 1.0, "t1": 3.0, "stream": 0, "kind": "LlmBwd"},
            {"t0": 5.0, "t1": 6.0, "stream": 0, "kind": "LlmFwd"}, {"t0": 3.0, "t1": 5.0, "stream": 1, "kind": "GenFwd"},
            {"t0": 4.0, "t1": 4.0, "stream": 0, "kind": "Recv"}, {"t0": 6.0, "t1": 8.0, "stream": 0, "kind": "Tail"}]
    frac, span = bench.bubble_from_trace(recs)
    assert span == 8.0 and abs(frac - 0.5) < 1e-12


def test_step_hbm_bytes_is_below_the_flop_term_at_c2():
    # the step roofline's HBM term (algorithmic bytes / measured HBM bandwidth) is
    # positive and, for this GEMM-dominated step, below the tensor-core term
    from synth import get_config
    cfg = get_config("C2", P=1, M=1)
    b = bench.step_hbm_bytes(cfg, [554], [554])
    f = bench.step_flops(cfg, [554], [554])
    assert b > 0
    assert b / 6555e9 < f / 1664.4e12
    # weights are read per microbatch: bytes grow linearly in M
    assert abs(bench.step_hbm_bytes(cfg, [554] * 4, [554] * 4) - 4 * b) < 1e-6 * b


def test_zb_h1_workload_and_bubble_bound():
    cfg, P, D = bench.workload(ns(llm_sched="zb_h1"), 4)
    assert (cfg.llm_sched, P, D, cfg.M) == ("zb_h1", 4, 1, 64)
    assert bench.bubble_bound(cfg, P) == pytest.approx(3 / (3 * 64 + 3))
    ref, _, _ = bench.workload(ns(), 4)
    assert bench.bubble_bound(ref, P) == pytest.approx(3 / 67)
    assert "ZB-H1" in bench.config_dict(cfg, P, D)["workload"]
    with pytest.raises(SystemExit):
        bench.workload(ns(config="C3", llm_sched="zb_h1"), 4)


def test_half_layer_unit_partition():
    """--partition halves (bigmac.h stage_halves, R24): 2L units split over P V stages,
    the slowest stage (A = 2/3, B = 1/3 layer, head on the last) minimised."""
    from synth import get_config
    cfg = get_config("C2", P=4, M=64)
    u = bench.unit_partition(cfg, 4)
    assert sum(u) == 2 * cfg.L and min(u) >= 1
    costs = bench.unit_costs(cfg, u)
    assert max(costs) < 5.0 - 1e-9                 # beats the best whole-layer split (4, 4, 5, 3)
    assert max(costs) == pytest.approx(14 / 3)
    # brute force over every 4-way split of the 32 units
    import itertools
    best = min(max(bench.unit_costs(cfg, [a, b - a, c - b, 32 - c]))
               for a, b, c in itertools.combinations(range(1, 32), 3))
    assert max(costs) == pytest.approx(best)
    assert bench.pacing_stage_mask(u, 4, costs) == 0b0101
    assert bench.lightest_only_mask(costs) == 0b0111          # encoder / generator on the last stage only
    a = ns(partition="halves", gen_exclude="auto", enc_exclude="auto", head="auto")
    assert bench.gen_exclude(a, cfg, 4, u, "bigmac") == 0b0111
    assert bench.enc_exclude(a, cfg, 4, u, "bigmac") == 0b0111     # slack 0.64 >= ENC_GEN_LAYERS
    c2 = get_config("C2", P=2, M=32)
    u2 = bench.unit_partition(c2, 2)
    assert bench.enc_exclude(a, c2, 2, u2, "bigmac") == 0           # slack 0.3: the encoder stays everywhere
    assert bench.gen_exclude(a, c2, 2, u2, "bigmac") == 0b01
    assert bench.pacing_stage_mask([4, 4, 5, 3], 4) == 0b0100
    assert bench.pacing_stage_mask([4, 4, 4, 4], 4) == 0
    a = ns(partition="halves", llm_sched="auto")
    assert bench.stage_split(a, cfg, 4) == u
    assert bench.stage_split(a, cfg.replace(P=1), 1) is None or cfg.V > 1
