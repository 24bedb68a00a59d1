"""GPU parity of the full nested-pipeline step (bm_step through the C ABI)
against the fp64 oracle: loss, per-microbatch loss terms and every parameter
gradient, normwise relative error <= 1e-4 (fp32) / 2e-2 (bf16) -- the
tolerances north_star fixes.  Single-GPU cases run the P = 1 pipeline; the
multi-rank cases (P = 2, 4, replicas) launch one process per rank via torchrun --
one per GPU when the box has enough GPUs, else all on cuda:0 (_torchrun)."""
import os
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from synth import get_config, make_batch, make_weights  # noqa: E402
from oracle import model as om  # noqa: E402

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOL = {"f32": 1e-4, "bf16": 2e-2}


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


@pytest.fixture(scope="module")
def oracle_cache():
    return {}


@pytest.fixture
def gemm_mode(request):
    """bm_k_gemm_mode for the test: 0 = auto (C1 sizes take the 1-CTA kernels),
    2 = CTA pairs everywhere -- the kernels the C2 / C4 bench runs for the LLM
    contractions (pair DSWIGLU down dgrad, pair reduce-add wgrad, pair residual add)."""
    from paper_2605_25451_b200 import _lib as L
    mode = getattr(request, "param", 0)
    L.call("bm_k_gemm_mode", mode)
    yield mode
    L.call("bm_k_gemm_mode", 0)


def reference(cache, cfg):
    key = (cfg.P, cfg.M, cfg.V, cfg.name)
    if key not in cache:
        W, B = make_weights(cfg), make_batch(cfg)
        cache[key] = (W, B, om.step_fp64(cfg, W, B))
    return cache[key]


@pytest.mark.parametrize("dtype,gemm_mode", [("f32", 0), ("bf16", 0), ("bf16", 2)], indirect=["gemm_mode"])
@pytest.mark.parametrize("M,V", [(4, 1), (4, 2), (1, 1), (6, 1)])
def test_step_single_gpu(oracle_cache, dtype, M, V, gemm_mode):
    from paper_2605_25451_b200.runtime import Runtime
    cfg = get_config("C1", P=1, M=M, V=V)
    W, B, (loss_ref, per_ref, G_ref) = reference(oracle_cache, cfg)
    rt = Runtime(cfg, dtype)
    rt.load_weights(W)
    db = rt.device_batch(B)
    rt.step(db)
    torch.cuda.synchronize()
    loss, ce, mse = rt.losses()
    tol = TOL[dtype]
    assert abs(loss - loss_ref) <= tol * abs(loss_ref)
    assert rel(ce, np.array([a for a, _ in per_ref])) <= tol
    assert rel(mse, np.array([b for _, b in per_ref])) <= tol
    worst = {}
    for name in rt.names():
        worst[name] = rel(rt.grad(name), G_ref[name])
    bad = {k: v for k, v in worst.items() if v > tol}
    assert not bad, bad
    # determinism: a second step reproduces every gradient bit for bit
    g1 = rt.grads_t.clone()
    rt.step(db)
    torch.cuda.synchronize()
    assert torch.equal(g1, rt.grads_t)
    # the end-to-end path (host batch copied in inside the step) gives the same result
    hb = rt.host_batch(B)
    rt.step(hb)
    torch.cuda.synchronize()
    assert torch.equal(g1, rt.grads_t)
    assert rt.launch_count() > 0
    rt.close()


@pytest.mark.parametrize("kw", [{"enc_place": "entry_stage", "gen_place": "last_stage"}, {"warmup_units": 4},
                                {"warmup_units": 2}])
def test_step_single_gpu_baselines(oracle_cache, kw):
    from paper_2605_25451_b200.runtime import Runtime
    cfg = get_config("C1", P=1, M=4, V=1)
    W, B, (loss_ref, per_ref, G_ref) = reference(oracle_cache, cfg)
    rt = Runtime(cfg, "f32", sched_kw=kw)
    rt.load_weights(W)
    rt.step(rt.device_batch(B))
    torch.cuda.synchronize()
    loss, _, _ = rt.losses()
    assert abs(loss - loss_ref) <= 1e-4 * abs(loss_ref)
    bad = {n: rel(rt.grad(n), G_ref[n]) for n in rt.names()}
    assert not {k: v for k, v in bad.items() if v > 1e-4}
    rt.close()


@pytest.mark.parametrize("cfg_name,dtype", [("C1", "f32"), ("C1", "bf16"), ("C1M", "f32"), ("C1M", "bf16")])
def test_step_single_gpu_head_dp_shard(oracle_cache, cfg_name, dtype):
    """BM_HEAD_DP_SHARD at P = 1: the LM head + CE run inside GenFwd on the
    generator stream (the single shard is the whole text range); same results."""
    from paper_2605_25451_b200.runtime import Runtime
    cfg = get_config(cfg_name, P=1, M=4, V=1)
    W, B, (loss_ref, per_ref, G_ref) = reference(oracle_cache, cfg)
    rt = Runtime(cfg, dtype, head_place="dp_shard")
    assert rt.params["llm.head"][4] == 0          # DP parameter
    rt.load_weights(W)
    db = rt.device_batch(B)
    rt.step(db)
    torch.cuda.synchronize()
    loss, ce, mse = rt.losses()
    tol = TOL[dtype]
    assert abs(loss - loss_ref) <= tol * abs(loss_ref)
    assert rel(ce, np.array([a for a, _ in per_ref])) <= tol
    bad = {n: rel(rt.grad(n), G_ref[n]) for n in rt.names()}
    assert not {k: v for k, v in bad.items() if v > tol}, bad
    g1 = rt.grads_t.clone()
    rt.step(db)
    torch.cuda.synchronize()
    assert torch.equal(g1, rt.grads_t)
    rt.close()


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_step_single_gpu_uneven_partition(oracle_cache, dtype):
    """last_stage_layers = 1 at P = 1, V = 2: virtual stages hold layers (3, 1)."""
    from paper_2605_25451_b200.runtime import Runtime
    cfg = get_config("C1", P=1, M=4, V=2)
    W, B, (loss_ref, per_ref, G_ref) = reference(oracle_cache, cfg)
    rt = Runtime(cfg, dtype, last_stage_layers=1)
    rt.load_weights(W)
    rt.step(rt.device_batch(B))
    torch.cuda.synchronize()
    loss, _, _ = rt.losses()
    tol = TOL[dtype]
    assert abs(loss - loss_ref) <= tol * abs(loss_ref)
    bad = {n: rel(rt.grad(n), G_ref[n]) for n in rt.names()}
    assert not {k: v for k, v in bad.items() if v > tol}, bad
    rt.close()


@pytest.mark.parametrize("cfg_name", ["C1", "C1M"])
@pytest.mark.parametrize("dtype,gemm_mode", [("f32", 0), ("bf16", 0), ("bf16", 2)], indirect=["gemm_mode"])
def test_step_edge_batches_single_gpu(cfg_name, dtype, gemm_mode):
    """Degenerate microbatches (synth.edge_counts): n_mod = 0, n_mod = S (no CE rows),
    generator rows spanning the sequence (overlapping modality and CE rows)."""
    from synth import edge_counts, edge_shape
    from paper_2605_25451_b200.runtime import Runtime
    cfg = edge_shape(get_config(cfg_name, P=1, M=4, V=1))
    n_mod, n_gen = edge_counts(cfg, 4)
    W, B = make_weights(cfg), make_batch(cfg, n_mod=n_mod, n_gen=n_gen)
    loss_ref, per_ref, G_ref = om.step_fp64(cfg, W, B)
    rt = Runtime(cfg, dtype)
    rt.load_weights(W)
    rt.step(rt.device_batch(B))
    torch.cuda.synchronize()
    loss, ce, mse = rt.losses()
    tol = TOL[dtype]
    assert abs(loss - loss_ref) <= tol * abs(loss_ref)
    assert ce[1] == 0.0   # n_mod = S: no CE rows
    assert rel(ce, np.array([a for a, _ in per_ref])) <= tol
    assert rel(mse, np.array([b for _, b in per_ref])) <= tol
    bad = {n: rel(rt.grad(n), G_ref[n]) for n in rt.names()}
    assert not {k: v for k, v in bad.items() if v > tol}, bad
    rt.close()


def test_trace_records_every_op():
    """bm_ctx_trace_get: one record per compute op / receive (+ the tail), in the
    rank's op order on each stream, with non-decreasing times; tracing does not
    change the step's results."""
    from paper_2605_25451_b200.runtime import Runtime
    cfg = get_config("C1", P=1, M=4, V=1)
    W, B = make_weights(cfg), make_batch(cfg)
    rt = Runtime(cfg, "f32")
    rt.load_weights(W)
    db = rt.device_batch(B)
    rt.step(db)
    torch.cuda.synchronize()
    loss0 = rt.losses()[0]
    rt.set_trace(True)
    rt.step(db)
    torch.cuda.synchronize()
    tr = rt.trace()
    rt.set_trace(False)
    ops = rt.sched.ops(0)
    n_compute = sum(1 for o in ops if o[0] <= 5)
    assert len(tr) == n_compute + 1
    assert tr[-1]["kind"] == "Tail"
    main = [x for x in tr if x["stream"] == 0 and x["kind"] != "Tail"]
    assert [x["op"] for x in main] == sorted(x["op"] for x in main)
    for a, b in zip(main, main[1:]):
        assert a["t0"] <= a["t1"] <= b["t0"] + 1e-3
    assert abs(rt.losses()[0] - loss0) <= 1e-6 * abs(loss0)
    rt.close()


@pytest.mark.parametrize("dtype,gemm_mode", [("f32", 0), ("bf16", 0), ("bf16", 2)], indirect=["gemm_mode"])
@pytest.mark.parametrize("M,V", [(4, 1), (4, 2)])
def test_step_single_gpu_medium(oracle_cache, dtype, M, V, gemm_mode):
    # C1M: several tiles per GEMM dimension, ragged row counts (60..200 modality rows)
    from paper_2605_25451_b200.runtime import Runtime
    cfg = get_config("C1M", P=1, M=M, V=V)
    W, B, (loss_ref, per_ref, G_ref) = reference(oracle_cache, cfg)
    rt = Runtime(cfg, dtype)
    rt.load_weights(W)
    rt.step(rt.device_batch(B))
    torch.cuda.synchronize()
    loss, ce, mse = rt.losses()
    tol = TOL[dtype]
    assert abs(loss - loss_ref) <= tol * abs(loss_ref)
    bad = {n: rel(rt.grad(n), G_ref[n]) for n in rt.names()}
    bad = {k: v for k, v in bad.items() if v > tol}
    assert not bad, bad
    rt.close()


@pytest.mark.parametrize("cfg_name,dtype,gemm_mode", [("C1", "f32", 0), ("C1", "bf16", 0), ("C1M", "f32", 0),
                                                     ("C1M", "bf16", 2)], indirect=["gemm_mode"])
def test_step_single_gpu_zb_h1(oracle_cache, cfg_name, dtype, gemm_mode):
    """ZB-H1 base schedule (reading R23) at P = 1: LLM_BWD computes only the input
    gradient and leaves dY / dgu per layer in the stash slot, LLM_W runs the weight
    gradient GEMMs -- same loss and gradients as the oracle."""
    from paper_2605_25451_b200.runtime import Runtime
    cfg = get_config(cfg_name, P=1, M=4, V=1)
    W, B, (loss_ref, per_ref, G_ref) = reference(oracle_cache, cfg)
    rt = Runtime(cfg, dtype, sched_kw={"llm_sched": "zb_h1"})
    assert any(o[0] == 8 for o in rt.sched.ops(0))          # BM_OP_LLM_W present
    rt.load_weights(W)
    db = rt.device_batch(B)
    rt.step(db)
    torch.cuda.synchronize()
    loss, ce, mse = rt.losses()
    tol = TOL[dtype]
    assert abs(loss - loss_ref) <= tol * abs(loss_ref)
    bad = {n: rel(rt.grad(n), G_ref[n]) for n in rt.names()}
    assert not {k: v for k, v in bad.items() if v > tol}, bad
    g1 = rt.grads_t.clone()
    rt.step(db)
    torch.cuda.synchronize()
    assert torch.equal(g1, rt.grads_t)
    rt.close()


def _torchrun(nproc, cases, timeout=900):
    """Launch mp_step.py on nproc ranks for a batch of cases.  With fewer GPUs than
    ranks every rank runs on cuda:0 (BM_TEST_ONE_GPU=1): stage-boundary copies,
    credit rings and gather / scatter handoffs go through CUDA IPC within the
    device, and the step-end sums through the library's peer-memory reduce (NCCL
    rejects duplicate GPUs), so the cross-rank half of the step is verified on a
    1-GPU box too.  Returns {case: result line}."""
    e = dict(os.environ)
    if torch.cuda.device_count() < nproc:
        e["BM_TEST_ONE_GPU"] = "1"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", "--master-port", str(29500 + nproc), os.path.join(ROOT, "tests", "mp_step.py"),
           *cases]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=ROOT, env=e)
    out = {}
    for line in r.stdout.splitlines():
        if line.startswith("CASE "):
            parts = line.split(" ", 2)
            out[parts[1]] = parts[2]
    out["__tail__"] = r.stdout[-3000:] + r.stderr[-3000:]
    return out


# (config, P, M, V, dtype, spec, D, flags): mp_step.py's case grammar
MR_CASES = [
    # 1F1B / interleaved, both dtypes, DP-sharded and last-stage generator
    ("C1", 2, 4, 1, "f32", "dp_shard", 1, ""), ("C1", 2, 4, 1, "bf16", "dp_shard", 1, ""),
    ("C1", 2, 8, 2, "f32", "dp_shard", 1, ""), ("C1", 2, 4, 1, "f32", "last_stage", 1, ""),
    ("C1M", 2, 4, 1, "bf16", "dp_shard", 1, ""), ("C1M", 2, 4, 2, "f32", "dp_shard", 1, ""),
    # placement knobs: DP-sharded head (R14), uneven / explicit partitions (R16)
    ("C1", 2, 4, 1, "f32", "dp_shard+head_dp", 1, ""), ("C1", 2, 8, 2, "bf16", "dp_shard+head_dp", 1, ""),
    ("C1", 2, 4, 1, "f32", "dp_shard+last1", 1, ""), ("C1", 2, 4, 1, "bf16", "dp_shard+last3", 1, ""),
    ("C1", 2, 4, 1, "f32", "dp_shard+split1-3", 1, ""),
    # the paper's baselines on the same executor (f1): memory- and compute-efficient
    ("C1", 2, 4, 1, "f32", "entry_stage+last_stage", 1, ""), ("C1", 2, 4, 1, "bf16", "ce", 1, ""),
    # degenerate batches
    ("C1", 2, 4, 1, "bf16", "dp_shard+edge", 1, ""), ("C1", 2, 8, 2, "f32", "dp_shard+edge", 1, ""),
    # every bf16 contraction on the CTA-pair GEMM (the bench's LLM kernels)
    ("C1M", 2, 4, 1, "bf16", "dp_shard", 1, "gm2"), ("C1M", 2, 8, 2, "bf16", "dp_shard", 1, "gm2"),
    # FSDP: one-sided pull (also with the last-stage generator), all-gather baseline
    ("C1", 2, 4, 1, "f32", "dp_shard+fsdp", 1, ""), ("C1", 2, 8, 2, "bf16", "dp_shard+fsdp", 1, ""),
    ("C1", 2, 4, 1, "f32", "last_stage+fsdp", 1, ""), ("C1", 2, 4, 1, "f32", "dp_shard+fsdpag", 1, ""),
    ("C1M", 2, 4, 1, "bf16", "dp_shard+fsdp", 1, "gm2"), ("C1", 2, 4, 1, "f32", "dp_shard+genx2", 1, ""),
    ("C1", 2, 8, 2, "f32", "dp_shard+encx2", 1, ""), ("C1", 2, 4, 1, "bf16", "dp_shard+encx1+edge", 1, ""),
    # pipeline replicas (R15)
    ("C1", 1, 4, 1, "f32", "dp_shard", 2, ""), ("C1", 1, 4, 1, "bf16", "dp_shard", 2, ""),
    # the peer-memory step-end sum forced (also where NCCL would be used)
    ("C1", 2, 4, 1, "f32", "dp_shard", 1, "peer"),
    # P = 4
    ("C1", 4, 8, 1, "f32", "dp_shard", 1, ""), ("C1", 4, 8, 1, "bf16", "dp_shard", 1, ""),
    ("C1", 4, 16, 1, "bf16", "dp_shard", 1, ""), ("C1", 4, 16, 1, "bf16", "ce", 1, ""),
    ("C1", 4, 16, 1, "f32", "entry_stage+last_stage", 1, ""), ("C1", 4, 16, 1, "f32", "ce", 1, ""),
    ("C1", 4, 8, 1, "bf16", "dp_shard+head_dp", 1, ""), ("C1", 4, 4, 1, "f32", "dp_shard+edge", 1, ""),
    ("C1", 4, 8, 1, "bf16", "dp_shard+edge", 1, ""), ("C1", 4, 8, 1, "bf16", "last_stage+edge", 1, ""),
    ("C1M", 4, 8, 1, "bf16", "dp_shard", 1, "gm2"),
    # generator rows kept off a rank (bigmac.h gen_exclude, reading R20)
    ("C1", 4, 8, 1, "f32", "dp_shard+genx4", 1, ""), ("C1", 4, 8, 1, "bf16", "dp_shard+genx9+edge", 1, ""),
    # encoder microbatches moved off ranks (bm_sched_cfg.enc_exclude, reading R22)
    ("C1", 4, 8, 1, "f32", "dp_shard+encx4", 1, ""), ("C1", 4, 8, 1, "bf16", "dp_shard+encx4+genx4", 1, ""),
    ("C1", 4, 8, 1, "f32", "dp_shard+encx1", 1, ""), ("C1M", 4, 8, 1, "bf16", "dp_shard+encx6+fsdp", 1, ""),
    # FSDP of the encoder / generator: one-sided pull, and the all-gather baseline
    ("C1", 4, 8, 1, "f32", "dp_shard+fsdpag", 1, ""), ("C1M", 4, 8, 1, "bf16", "dp_shard+fsdp", 1, ""),
    ("C1", 4, 8, 1, "f32", "dp_shard+fsdp", 1, ""),
    # ZB-H1 zero-bubble base schedule (B = input gradient, W = weight gradients; R23)
    ("C1", 2, 4, 1, "f32", "dp_shard+zb", 1, ""), ("C1", 2, 4, 1, "bf16", "dp_shard+zb", 1, ""),
    ("C1M", 2, 4, 1, "bf16", "dp_shard+zb", 1, "gm2"), ("C1", 2, 4, 1, "f32", "entry_stage+last_stage+zb", 1, ""),
    ("C1", 4, 8, 1, "f32", "dp_shard+zb", 1, ""), ("C1", 4, 16, 1, "bf16", "dp_shard+zb", 1, ""),
    ("C1", 4, 8, 1, "f32", "last_stage+zb+edge", 1, ""), ("C1M", 4, 8, 1, "bf16", "dp_shard+zb+fsdp", 1, "gm2"),
    ("C1", 2, 4, 1, "f32", "dp_shard+zb", 2, ""),
    # stage boundaries inside layers (half-layer units, R24): [x | h] / [dx | dh] messages
    ("C1", 2, 4, 1, "f32", "dp_shard+halves3-5", 1, ""), ("C1", 2, 4, 1, "bf16", "dp_shard+halves5-3", 1, ""),
    ("C1M", 2, 4, 1, "bf16", "dp_shard+halves3-5", 1, "gm2"), ("C1", 2, 4, 1, "f32", "dp_shard+halves3-5+zb", 1, ""),
    ("C1", 2, 8, 2, "f32", "dp_shard+halves1-3-2-2", 1, ""), ("C1", 4, 8, 1, "f32", "dp_shard+halves3-2-2-1", 1, ""),
    ("C1", 4, 8, 1, "bf16", "dp_shard+halves1-1-1-5+zb+edge", 1, ""), ("C1", 2, 4, 1, "f32", "dp_shard+halves3-5", 2, ""),
    # the bench's multi-GPU defaults: half-layer units, generator / encoder on the lightest stage (N = 4, and
    # N = 8 as P = 4 x D = 2 -- here P = 2 x D = 2), 1F1B and ZB-H1
    ("C1", 4, 8, 1, "bf16", "dp_shard+halves3-2-2-1+genx7+encx7", 1, "es"),
    ("C1", 4, 8, 1, "f32", "dp_shard+halves3-2-2-1+genx7+encx7+zb", 1, ""),
    ("C1", 2, 4, 1, "bf16", "dp_shard+halves5-3+genx1+encx1", 2, ""),
    # the N = 8 bench shape: P = 4 stages x D = 2 replicas (world 8), half-layer units,
    # encoder / generator on the lightest stage
    ("C1", 4, 8, 1, "bf16", "dp_shard+halves3-2-2-1+genx7+encx7", 2, "es"),
    ("C1", 2, 4, 1, "f32", "dp_shard+encx1", 1, "es"), ("C1", 4, 8, 1, "f32", "dp_shard+halves3-2-2-1+genx7+encx7+zb", 1, "es"),
    ("C1", 4, 8, 1, "f32", "dp_shard+halves3-2-2-1+genx7+encx7+zb", 2, ""),
    # P = 2 x D = 2
    ("C1", 2, 4, 1, "f32", "dp_shard", 2, ""), ("C1", 2, 4, 1, "bf16", "dp_shard", 2, ""),
    ("C1", 2, 8, 2, "f32", "dp_shard", 2, ""), ("C1", 2, 4, 1, "f32", "dp_shard", 2, "peer"),
    ("C1M", 2, 4, 1, "bf16", "dp_shard", 2, "gm2"),
]


def _case_str(c):
    return ":".join(map(str, c))


_MR_RESULTS = {}


def _mr_result(case):
    """Run every case of this world size in one torchrun launch (once), return this case's line."""
    world = case[1] * case[6]
    if world not in _MR_RESULTS:
        cases = [_case_str(c) for c in MR_CASES if c[1] * c[6] == world]
        _MR_RESULTS[world] = _torchrun(world, cases)
    res = _MR_RESULTS[world]
    return res.get(_case_str(case)), res["__tail__"]


@pytest.mark.parametrize("case", MR_CASES, ids=_case_str)
def test_step_multirank(case):
    """The nested-pipeline step across ranks vs the fp64 oracle: stage-boundary act /
    grad rings (A11 / A15), encoder gather / embgrad scatter (A8 / A16), generator
    scatter / gather (A13), step-end DP / replica sums (A18)."""
    line, tail = _mr_result(case)
    assert line is not None, tail
    assert "PARITY OK" in line, line
    if "peer" in case[7]:
        assert "sum_mode peer" in line, line


def test_step_wait_timeout_names_blocked_op():
    """A rank whose peer stops stepping does not hang the caller: bm_step_wait returns
    BM_E_TIMEOUT naming the first unmet receive / credit wait (P:362-363 waits on
    receive handles; SURVEY §8(b) flag-wait timeout)."""
    out = _torchrun(2, ["hang"], timeout=300)
    assert "TIMEOUT OK" in out.get("hang", ""), out


@pytest.mark.parametrize("fsdp,dtype", [("pull", "f32"), ("pull", "bf16"), ("allgather", "f32")])
def test_step_single_gpu_fsdp(oracle_cache, fsdp, dtype):
    """FSDP at P = 1 (the shard is everything): the bucket chain (two slots per chain,
    pulls on the pull stream, parameter lookups into the acquired block) reproduces
    the plain step."""
    from paper_2605_25451_b200.runtime import Runtime
    cfg = get_config("C1M", P=1, M=4, V=1)
    W, B, (loss_ref, per_ref, G_ref) = reference(oracle_cache, cfg)
    rt = Runtime(cfg, dtype, fsdp=fsdp)
    rt.load_weights(W)
    rt.step(rt.device_batch(B))
    torch.cuda.synchronize()
    loss, _, _ = rt.losses()
    tol = TOL[dtype]
    assert abs(loss - loss_ref) <= tol * abs(loss_ref)
    bad = {n: rel(rt.grad(n), G_ref[n]) for n in rt.names()}
    assert not {k: v for k, v in bad.items() if v > tol}, bad
    rt.close()
