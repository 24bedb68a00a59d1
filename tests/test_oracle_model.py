"""Pins for the numeric oracle (O-N): closed forms, finite differences, an
independent autograd cross-check (library used only as a pin), and the
schedule interpreter against the sequential definition."""
import numpy as np
import pytest

from synth import get_config, make_batch, make_weights
from oracle import model as om
from oracle import interp
from oracle import schedule as S


@pytest.fixture(scope="module")
def tiny():
    cfg = get_config("C1", M=2, P=1)
    return cfg, make_weights(cfg), make_batch(cfg)


def test_zero_head_gives_log_vocab(tiny):
    # CE over a uniform softmax = log(vocab) exactly (definition of cross-entropy)
    cfg, W, B = tiny
    W = dict(W)
    W["llm.head"] = np.zeros_like(W["llm.head"])
    _, per, _ = om.step_fp64(cfg, W, B)
    for ce, _ in per:
        assert abs(ce - np.log(cfg.vocab)) < 1e-12


def test_zero_generator_out_gives_mean_square_target(tiny):
    # out = 0 => MSE = mean(t^2) over the full microbatch (SURVEY Q9 denominator)
    cfg, W, B = tiny
    W = dict(W)
    W["gen.out"] = np.zeros_like(W["gen.out"])
    _, per, _ = om.step_fp64(cfg, W, B)
    for m, (_, mse) in enumerate(per):
        t = np.asarray(B.targets[m], np.float64)
        assert abs(mse - np.mean(t * t)) < 1e-12


def test_zero_down_makes_llm_identity(tiny):
    cfg, W, B = tiny
    W = {k: np.asarray(v, np.float64) for k, v in W.items()}
    for l in range(cfg.L):
        W[f"llm.layer{l}.down"] = np.zeros_like(W[f"llm.layer{l}.down"])
    x = np.random.default_rng(0).standard_normal((cfg.S, cfg.d))
    y, _ = om.llm_layers_fwd(W, cfg, list(range(cfg.L)), x)
    assert np.array_equal(y, x)


def test_embed_rows(tiny):
    # P:297 embed_preprocess: text rows come from the table, modality rows from the encoder
    cfg, W, B = tiny
    W = om.to_f64(W)
    n = int(B.n_mod[0])
    emb = np.full((n, cfg.d), 7.0)
    X = om.embed_fwd(W, B.ids[0], emb, n)
    assert np.array_equal(X[:n], emb)
    assert np.array_equal(X[n:], W["llm.embed"][B.ids[0][n:]])


def test_rmsnorm_unit_rms():
    x = np.random.default_rng(1).standard_normal((16, 64)) * 3
    y, _ = om.rmsnorm(x, np.ones(64))
    rms = np.sqrt(np.mean(y * y, axis=1))
    assert np.allclose(rms, 1.0 / np.sqrt(1 + om.EPS / np.mean(x * x, axis=1)), rtol=0, atol=1e-12)


def test_gelu_tanh_close_to_erf_gelu():
    from scipy.special import erf
    a = np.linspace(-6, 6, 2001)
    exact = 0.5 * a * (1 + erf(a / np.sqrt(2)))
    assert np.max(np.abs(om.gelu(a) - exact)) < 1e-3
    assert om.gelu(np.zeros(1))[0] == 0.0


def test_swiglu_limits():
    f = 4
    gu = np.concatenate([np.array([[0.0, 40.0, -40.0, 1.0]]), np.array([[3.0, 2.0, 5.0, 1.0]])], axis=1)
    h = om.swiglu(gu, f)
    assert h[0, 0] == 0.0
    assert abs(h[0, 1] - 80.0) < 1e-12
    assert abs(h[0, 2]) < 1e-12
    assert abs(h[0, 3] - 1.0 / (1.0 + np.exp(-1.0))) < 1e-15


def test_finite_differences_per_tensor(tiny):
    # central differences; directional derivative along a random direction per
    # tensor, relative error <= 1e-6 above the fp64 roundoff floor
    cfg, W, B = tiny
    loss, _, G = om.step_fp64(cfg, W, B)
    W64 = om.to_f64(W)
    rng = np.random.default_rng(3)
    h = 1e-5
    for name in sorted(W64):
        v = rng.standard_normal(W64[name].shape)
        v /= np.linalg.norm(v)
        Wp = dict(W64); Wp[name] = W64[name] + h * v
        Wm = dict(W64); Wm[name] = W64[name] - h * v
        fd = (om.loss_only(cfg, Wp, B) - om.loss_only(cfg, Wm, B)) / (2 * h)
        an = float(np.sum(G[name] * v))
        # roundoff floor of the difference quotient: ~100 eps |L| / h
        assert abs(fd - an) <= 1e-6 * abs(an) + 100 * 2.2e-16 * abs(loss) / h, (name, fd, an)


def test_autograd_crosscheck(tiny):
    # independent formulation in torch float64 with autograd (library used as a pin only)
    torch = pytest.importorskip("torch")
    cfg, W, B = tiny
    loss_ref, _, G = om.step_fp64(cfg, W, B)
    T = {k: torch.tensor(np.asarray(v, np.float64), requires_grad=True) for k, v in W.items()}
    F = torch.nn.functional

    def rms(x, g):
        return x * torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + om.EPS) * g

    def blk(x, p):
        return x + F.linear(F.gelu(F.linear(rms(x, T[p + ".norm"]), T[p + ".fc1"]), approximate="tanh"),
                            T[p + ".fc2"])

    M = len(B.n_mod)
    total = 0
    for m in range(M):
        n_mod, n_gen = int(B.n_mod[m]), int(B.n_gen[m])
        e = F.linear(torch.tensor(np.asarray(B.patches[m], np.float64)), T["enc.patch"])
        for i in range(cfg.L_e):
            e = blk(e, f"enc.blk{i}")
        e = F.linear(F.gelu(F.linear(e, T["enc.proj1"]), approximate="tanh"), T["enc.proj2"])
        ids = torch.tensor(B.ids[m].astype(np.int64))
        x = torch.cat([e, T["llm.embed"][ids[n_mod:]]], 0)
        for l in range(cfg.L):
            p = f"llm.layer{l}"
            gu = F.linear(rms(x, T[p + ".norm"]), T[p + ".gate_up"])
            x = x + F.linear(F.silu(gu[:, :cfg.f]) * gu[:, cfg.f:], T[p + ".down"])
        hn = rms(x, T["llm.final_norm"])
        ce = F.cross_entropy(F.linear(hn[n_mod:], T["llm.head"]),
                             torch.tensor(B.labels[m][n_mod:].astype(np.int64)))
        g = F.linear(hn[cfg.S - n_gen:], T["gen.in"])
        for i in range(cfg.L_g):
            g = blk(g, f"gen.blk{i}")
        mse = F.mse_loss(F.linear(g, T["gen.out"]), torch.tensor(np.asarray(B.targets[m], np.float64)))
        total = total + ce + mse
    loss = total / M
    loss.backward()
    assert abs(loss.item() - loss_ref) < 1e-12
    for k in T:
        ref = T[k].grad.numpy()
        assert np.linalg.norm(G[k] - ref) <= 1e-10 * max(np.linalg.norm(ref), 1e-30), k


@pytest.mark.parametrize("P,M,V,gen", [(1, 4, 1, "dp_shard"), (2, 4, 1, "dp_shard"), (2, 4, 1, "last_stage"),
                                       (4, 4, 1, "dp_shard"), (2, 4, 2, "dp_shard"), (2, 8, 2, "dp_shard"),
                                       (1, 4, 2, "dp_shard")])
def test_interpreter_matches_sequential(P, M, V, gen):
    # S:424 / P:518: any valid schedule reaches the sequential gradients up to fp64 order
    cfg = get_config("C1", P=P, M=M, V=V)
    W, B = make_weights(cfg), make_batch(cfg)
    loss, per, G = om.step_fp64(cfg, W, B)
    sched = S.build(S.SchedCfg(P, M, V, llm_sched=cfg.llm_sched, gen_place=gen))
    loss2, per2, G2, _ = interp.run(sched, cfg, W, B)
    assert abs(loss2 - loss) <= 1e-12 * abs(loss)
    for k in G:
        assert np.linalg.norm(G2[k] - G[k]) <= 1e-12 * max(np.linalg.norm(G[k]), 1e-30), k
    # per-microbatch CE identical bitwise (forward is order independent)
    assert [a for a, _ in per] == [a for a, _ in per2]


@pytest.mark.parametrize("P,M,V,enc,gen,W", [(2, 4, 1, "entry_stage", "last_stage", 0), (2, 4, 1, "entry_stage", "dp_shard", 0),
                                             (4, 8, 1, "dp_unit", "dp_shard", 2), (2, 8, 2, "entry_stage", "last_stage", 0)])
def test_interpreter_baseline_strategies(P, M, V, enc, gen, W):
    # the baselines (memory-efficient entry-stage encoder, compute-efficient W = M/P)
    # reach the same gradients as the sequential definition
    cfg = get_config("C1", P=P, M=M, V=V)
    Wt, B = make_weights(cfg), make_batch(cfg)
    loss, per, G = om.step_fp64(cfg, Wt, B)
    sched = S.build(S.SchedCfg(P, M, V, llm_sched=cfg.llm_sched, enc_place=enc, gen_place=gen,
                               warmup_units=W if W else 0))
    loss2, per2, G2, _ = interp.run(sched, cfg, Wt, B)
    assert abs(loss2 - loss) <= 1e-12 * abs(loss)
    for k in G:
        assert np.linalg.norm(G2[k] - G[k]) <= 1e-12 * max(np.linalg.norm(G[k]), 1e-30), k


@pytest.mark.parametrize("D", [2, 3])
def test_replica_global_batch_is_mean_of_replicas(D):
    """Reading R15 (pipeline replicas): D replicas of M microbatches each compute
    the global-batch step.  L over the M*D-microbatch batch equals the mean of the
    D replica losses, and every gradient the mean of the replica gradients -- the
    sum the GPU path forms with scale 1/(M D) and an allreduce over replicas."""
    from synth import slice_batch
    M = 2
    cfg_g = get_config("C1", P=1, M=M * D, V=1)
    W, Bg = make_weights(cfg_g), make_batch(cfg_g)
    Lg, per_g, Gg = om.step_fp64(cfg_g, W, Bg)
    Ls, Gs = [], []
    for k in range(D):
        Lk, per_k, Gk = om.step_fp64(get_config("C1", P=1, M=M, V=1), W, slice_batch(Bg, k * M, (k + 1) * M))
        assert per_k == per_g[k * M:(k + 1) * M]          # per-microbatch terms are the replica's own
        Ls.append(Lk)
        Gs.append(Gk)
    assert abs(Lg - np.mean(Ls)) <= 1e-12 * abs(Lg)
    for name in Gg:
        mean = sum(G[name] for G in Gs) / D
        assert np.allclose(Gg[name], mean, rtol=1e-10, atol=1e-14), name


@pytest.mark.parametrize("P", [2, 3, 4])
def test_head_dp_shards_reproduce_full_head(P):
    """Reading R14 (DP-sharded LM head): text rows split into P shards
    [n_mod + floor(r n_text / P), n_mod + floor((r+1) n_text / P)); each shard's CE
    mean scaled by n_shard / n_text (the full-microbatch denominator) sums to the
    full CE, and each shard's dHn rows and head gradient (dce = n_shard / n_text)
    reassemble the unsharded backward exactly (up to fp64 rounding)."""
    cfg = get_config("C1", P=1, M=1, V=1)
    W = om.to_f64(make_weights(cfg))
    rng = np.random.default_rng(7)
    S, n_mod = cfg.S, 37
    H = rng.standard_normal((S, cfg.d))
    labels = rng.integers(0, cfg.vocab, size=S)
    Hn, ce, cache = om.head_fwd(W, cfg, H, labels, n_mod)
    G_full = {}
    dHn_full = om.head_bwd_logits(W, cfg, cache, 1.0, G_full)
    n_text = S - n_mod
    ce_sum, G_sh, dHn_sh = 0.0, {}, np.zeros_like(dHn_full)
    for r in range(P):
        lo = n_mod + (r * n_text) // P
        hi = n_mod + ((r + 1) * n_text) // P
        _, ce_r, cache_r = om.head_fwd(W, cfg, H[:hi], labels[:hi], lo)   # CE mean over rows [lo, hi)
        ce_sum += ce_r * (hi - lo) / n_text
        d = om.head_bwd_logits(W, cfg, cache_r, (hi - lo) / n_text, G_sh)
        dHn_sh[lo:hi] = d[lo:hi]
    assert abs(ce_sum - ce) <= 1e-12 * abs(ce)
    assert np.allclose(dHn_sh, dHn_full, rtol=1e-12, atol=1e-15)
    assert np.allclose(G_sh["llm.head"], G_full["llm.head"], rtol=1e-10, atol=1e-15)
