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


def _torchrun(nproc, *args, timeout=600, env=None):
    """Launch mp_step.py on nproc ranks.  With fewer GPUs than ranks every rank runs
    on cuda:0 (BM_TEST_ONE_GPU=1): stage-boundary copies, credit rings, gather /
    scatter handoffs go through CUDA IPC within the device, and the step-end sums
    through the library's peer-memory reduce (NCCL rejects duplicate GPUs), so the
    cross-rank half of the step is verified on a 1-GPU box too."""
    e = dict(os.environ)
    if torch.cuda.device_count() < nproc:
        e["BM_TEST_ONE_GPU"] = "1"
    e.update(env or {})
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", "--master-port", str(29500 + nproc), os.path.join(ROOT, "tests", "mp_step.py"),
           *map(str, args)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=ROOT, env=e)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]
    return r.stdout


@pytest.mark.parametrize("P,M,V,dtype,gen", [(2, 4, 1, "f32", "dp_shard"), (2, 4, 1, "bf16", "dp_shard"),
                                           (2, 8, 2, "f32", "dp_shard"), (2, 4, 1, "f32", "last_stage"),
                                           (2, 4, 1, "f32", "dp_shard+head_dp"), (2, 8, 2, "bf16", "dp_shard+head_dp"),
                                           (2, 4, 1, "f32", "dp_shard+last1"), (2, 4, 1, "bf16", "dp_shard+last3"), (2, 4, 1, "f32", "dp_shard+split1-3"),
                                           (2, 4, 1, "f32", "entry_stage+last_stage"),
                                           (2, 4, 1, "bf16", "ce"), (2, 4, 1, "bf16", "dp_shard+edge"),
                                           (2, 8, 2, "f32", "dp_shard+edge")])
def test_step_two_gpus(P, M, V, dtype, gen):
    out = _torchrun(P, "C1", P, M, V, dtype, gen)
    assert "PARITY OK" in out, out


@pytest.mark.parametrize("cfg_name,P,M,V,dtype", [("C1M", 2, 4, 1, "bf16"), ("C1M", 2, 4, 2, "f32")])
def test_step_two_gpus_medium(cfg_name, P, M, V, dtype):
    out = _torchrun(P, cfg_name, P, M, V, dtype, "dp_shard")
    assert "PARITY OK" in out, out


@pytest.mark.parametrize("P,M,V,dtype,gen", [(4, 8, 1, "f32", "dp_shard"), (4, 8, 1, "bf16", "dp_shard"),
                                           (4, 16, 1, "bf16", "dp_shard"), (4, 16, 1, "bf16", "ce"),
                                           (4, 16, 1, "f32", "entry_stage+last_stage"), (4, 16, 1, "f32", "ce"),
                                           (4, 8, 1, "bf16", "dp_shard+head_dp"), (4, 4, 1, "f32", "dp_shard+edge"),
                                           (4, 8, 1, "bf16", "dp_shard+edge"), (4, 8, 1, "bf16", "last_stage+edge")])
def test_step_four_gpus(P, M, V, dtype, gen):
    # "ce" (W = M / P) once deadlocked: a copy-engine send parked on a credit wait
    # blocked another stream's copy in a shared copy channel
    out = _torchrun(P, "C1", P, M, V, dtype, gen, timeout=240)
    assert "PARITY OK" in out, out


@pytest.mark.parametrize("P,D,M,V,dtype", [(1, 2, 4, 1, "f32"), (1, 2, 4, 1, "bf16")])
def test_step_replicas_two_gpus(P, D, M, V, dtype):
    # D pipeline replicas: DP params over all processes, LLM params per stage
    out = _torchrun(P * D, "C1", P, M, V, dtype, "dp_shard", D)
    assert "PARITY OK" in out, out


@pytest.mark.parametrize("P,D,M,V,dtype", [(2, 2, 4, 1, "f32"), (2, 2, 4, 1, "bf16"), (2, 2, 8, 2, "f32")])
def test_step_replicas_four_gpus(P, D, M, V, dtype):
    out = _torchrun(P * D, "C1", P, M, V, dtype, "dp_shard", D, timeout=300)
    assert "PARITY OK" in out, out


@pytest.mark.parametrize("P,D,M,V,dtype,gen", [(2, 1, 4, 1, "f32", "dp_shard"), (2, 2, 4, 1, "f32", "dp_shard")])
def test_step_peer_sum_forced(P, D, M, V, dtype, gen):
    """The library's peer-memory step-end sum (bm_ctx_init_peer_sum) also on
    distinct GPUs (BM_STEP_SUM=peer), where NCCL would otherwise be used."""
    out = _torchrun(P * D, "C1", P, M, V, dtype, gen, D, env={"BM_STEP_SUM": "peer"})
    assert "PARITY OK" in out and "sum_mode peer" in out, out


@pytest.mark.parametrize("P,D,M,V,dtype", [(2, 1, 4, 1, "bf16"), (2, 1, 8, 2, "bf16"), (2, 2, 4, 1, "bf16")])
def test_step_multirank_cta_pairs(P, D, M, V, dtype):
    """BM_GEMM_MODE=2: every bf16 contraction on the CTA-pair kernel (the bench's
    LLM path) across the stage boundaries and replicas."""
    out = _torchrun(P * D, "C1M", P, M, V, dtype, "dp_shard", D, env={"BM_GEMM_MODE": "2"})
    assert "PARITY OK" in out, out
