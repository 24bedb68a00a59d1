"""O-N: plain fp64 forward/backward of the synthetic MLLM (TEST INFRASTRUCTURE).

The method changes only WHEN and WHERE the model's work runs; the result it
reaches is the plain gradient of L = (1/M) sum_m (CE_m + MSE_m) accumulated
sequentially over microbatches ("changes only the order in which module
gradients are accumulated").  This file writes that
definition out with manual backprop in numpy float64.

Model:
  encoder   E0 = patches W_patch^T ; L_e x [E += fc2(gelu(fc1(rmsnorm(E))))]
            projector  Eout = proj2(gelu(proj1(E)))
  embed     X[i] = table[ids[i]] for i >= n_mod, X[:n_mod] = Eout
  LLM       L x [x += down(silu(g) * u)],  [g|u] = gate_up(rmsnorm(x))
  head      Hn = rmsnorm_final(H); CE = mean_{i in [n_mod,S)} -log softmax(Hn_i W_head^T)[label_i]
  generator Xg = Hn[S-n_gen:S]; G0 = Xg W_in^T; L_g x [G += fc2(gelu(fc1(rmsnorm(G))))];
            out = G W_out^T;  MSE = sum((out - t)^2) / (n_gen * d_t)
GELU is the tanh approximation; RMSNorm eps = 1e-5 (both fixed readings).
"""
from __future__ import annotations

import numpy as np

EPS = 1e-5
_C = np.sqrt(2.0 / np.pi)


# ----------------------------------------------------------------------------
# primitives (each with its own backward)
# ----------------------------------------------------------------------------
def rmsnorm(x, g):
    rstd = 1.0 / np.sqrt(np.mean(x * x, axis=-1, keepdims=True) + EPS)
    return x * rstd * g, rstd


def rmsnorm_bwd(dy, x, g, rstd):
    xhat = x * rstd
    dg = np.sum(dy * xhat, axis=0)
    dxhat = dy * g
    dx = rstd * (dxhat - xhat * np.mean(dxhat * xhat, axis=-1, keepdims=True))
    return dx, dg


def gelu(a):
    return 0.5 * a * (1.0 + np.tanh(_C * (a + 0.044715 * a ** 3)))


def gelu_bwd(dz, a):
    t = np.tanh(_C * (a + 0.044715 * a ** 3))
    return dz * (0.5 * (1.0 + t) + 0.5 * a * (1.0 - t * t) * _C * (1.0 + 3 * 0.044715 * a * a))


def swiglu(gu, f):
    g, u = gu[:, :f], gu[:, f:]
    s = 1.0 / (1.0 + np.exp(-g))
    return g * s * u


def swiglu_bwd(dh, gu, f):
    g, u = gu[:, :f], gu[:, f:]
    s = 1.0 / (1.0 + np.exp(-g))
    dg = dh * u * s * (1.0 + g * (1.0 - s))
    du = dh * g * s
    return np.concatenate([dg, du], axis=1)


def _acc(G, name, val):
    if name in G:
        G[name] = G[name] + val
    else:
        G[name] = np.array(val, dtype=np.float64)


# ----------------------------------------------------------------------------
# residual MLP block (encoder / generator): x + fc2(gelu(fc1(rmsnorm(x))))
# ----------------------------------------------------------------------------
def mlp_block_fwd(W, p, x):
    xn, rstd = rmsnorm(x, W[p + ".norm"])
    a = xn @ W[p + ".fc1"].T
    z = gelu(a)
    y = x + z @ W[p + ".fc2"].T
    return y, (x, xn, rstd, a, z)


def mlp_block_bwd(W, p, cache, dy, G):
    x, xn, rstd, a, z = cache
    _acc(G, p + ".fc2", dy.T @ z)
    dz = dy @ W[p + ".fc2"]
    da = gelu_bwd(dz, a)
    _acc(G, p + ".fc1", da.T @ xn)
    dxn = da @ W[p + ".fc1"]
    dx, dg = rmsnorm_bwd(dxn, x, W[p + ".norm"], rstd)
    _acc(G, p + ".norm", dg)
    return dy + dx


# ----------------------------------------------------------------------------
# encoder + projector (EncFwd / EncBwd of one microbatch)
# ----------------------------------------------------------------------------
def encoder_fwd(W, cfg, patches):
    caches = []
    e = patches @ W["enc.patch"].T
    for i in range(cfg.L_e):
        e, c = mlp_block_fwd(W, f"enc.blk{i}", e)
        caches.append(c)
    a1 = e @ W["enc.proj1"].T
    p1 = gelu(a1)
    out = p1 @ W["enc.proj2"].T
    return out, (patches, caches, e, a1, p1)


def encoder_bwd(W, cfg, cache, dout, G):
    patches, caches, e, a1, p1 = cache
    _acc(G, "enc.proj2", dout.T @ p1)
    dp1 = dout @ W["enc.proj2"]
    da1 = gelu_bwd(dp1, a1)
    _acc(G, "enc.proj1", da1.T @ e)
    de = da1 @ W["enc.proj1"]
    for i in reversed(range(cfg.L_e)):
        de = mlp_block_bwd(W, f"enc.blk{i}", caches[i], de, G)
    _acc(G, "enc.patch", de.T @ patches)


# ----------------------------------------------------------------------------
# embed_preprocess
# ----------------------------------------------------------------------------
def embed_fwd(W, ids, emb, n_mod):
    X = W["llm.embed"][ids].copy()
    X[:n_mod] = emb
    return X


def embed_bwd(cfg, dX, ids, n_mod, G):
    """Returns the modality-row gradient; accumulates the text-table gradient."""
    dT = np.zeros((cfg.vocab, cfg.d))
    for i in range(n_mod, dX.shape[0]):
        dT[ids[i]] += dX[i]
    _acc(G, "llm.embed", dT)
    return dX[:n_mod].copy()


# ----------------------------------------------------------------------------
# LLM layers (one virtual stage = a contiguous layer range)
# ----------------------------------------------------------------------------
def stage_layers(cfg, s):
    lps = cfg.L // (cfg.P * cfg.V)
    return list(range(s * lps, (s + 1) * lps))


def llm_layers_fwd(W, cfg, layers, x):
    caches = []
    for l in layers:
        p = f"llm.layer{l}"
        xn, rstd = rmsnorm(x, W[p + ".norm"])
        gu = xn @ W[p + ".gate_up"].T
        h = swiglu(gu, cfg.f)
        y = x + h @ W[p + ".down"].T
        caches.append((x, xn, rstd, gu, h))
        x = y
    return x, caches


def llm_layers_bwd(W, cfg, layers, caches, dy, G, defer=None):
    """Backward of llm_layers_fwd.  With `defer` (a list; zero-bubble B/W split,
    DESIGN.md R23) the two weight-gradient products dY^T X are appended to it as
    (name, dY, X) instead of accumulated; llm_wgrad applies them later."""
    def wgrad(name, dY, X):
        if defer is None:
            _acc(G, name, dY.T @ X)
        else:
            defer.append((name, dY, X))
    for l, c in zip(reversed(layers), reversed(caches)):
        p = f"llm.layer{l}"
        x, xn, rstd, gu, h = c
        wgrad(p + ".down", dy, h)
        dh = dy @ W[p + ".down"]
        dgu = swiglu_bwd(dh, gu, cfg.f)
        wgrad(p + ".gate_up", dgu, xn)
        dxn = dgu @ W[p + ".gate_up"]
        dx, dg = rmsnorm_bwd(dxn, x, W[p + ".norm"], rstd)
        _acc(G, p + ".norm", dg)
        dy = dy + dx
    return dy


def llm_wgrad(defer, G):
    """The W half of a zero-bubble backward: the deferred dY^T X products."""
    for name, dY, X in defer:
        _acc(G, name, dY.T @ X)


# ----------------------------------------------------------------------------
# last-stage head: final norm + LM head + CE over text rows
# ----------------------------------------------------------------------------
def head_fwd(W, cfg, H, labels, n_mod):
    Hn, rstd = rmsnorm(H, W["llm.final_norm"])
    z = Hn[n_mod:] @ W["llm.head"].T
    zmax = z.max(axis=1, keepdims=True)
    ez = np.exp(z - zmax)
    lse = np.log(ez.sum(axis=1, keepdims=True)) + zmax
    lab = labels[n_mod:]
    n_text = z.shape[0]
    ce = float(np.mean(lse[:, 0] - z[np.arange(n_text), lab])) if n_text else 0.0
    return Hn, ce, (H, Hn, rstd, z, lse, lab, n_mod)


def head_bwd_logits(W, cfg, cache, dce, G):
    """CE backward through the LM head: returns dHn (zero on modality rows)."""
    H, Hn, rstd, z, lse, lab, n_mod = cache
    n_text = z.shape[0]
    dHn = np.zeros_like(Hn)
    if n_text:
        p = np.exp(z - lse)
        p[np.arange(n_text), lab] -= 1.0
        dz = p * (dce / n_text)
        _acc(G, "llm.head", dz.T @ Hn[n_mod:])
        dHn[n_mod:] = dz @ W["llm.head"]
    return dHn


def final_norm_bwd(W, cache, dHn, G):
    H, Hn, rstd = cache[0], cache[1], cache[2]
    dH, dg = rmsnorm_bwd(dHn, H, W["llm.final_norm"], rstd)
    _acc(G, "llm.final_norm", dg)
    return dH


# ----------------------------------------------------------------------------
# generator on a row shard, MSE with the full-microbatch denominator (Q3, Q9)
# ----------------------------------------------------------------------------
def gen_fwd(W, cfg, X, t, denom):
    caches = []
    g = X @ W["gen.in"].T
    for i in range(cfg.L_g):
        g, c = mlp_block_fwd(W, f"gen.blk{i}", g)
        caches.append(c)
    out = g @ W["gen.out"].T
    diff = out - t
    mse_part = float(np.sum(diff * diff)) / denom
    return mse_part, (X, caches, g, diff, denom)


def gen_bwd(W, cfg, cache, dmse, G):
    X, caches, g, diff, denom = cache
    dout = diff * (2.0 * dmse / denom)
    _acc(G, "gen.out", dout.T @ g)
    dg = dout @ W["gen.out"]
    for i in reversed(range(cfg.L_g)):
        dg = mlp_block_bwd(W, f"gen.blk{i}", caches[i], dg, G)
    _acc(G, "gen.in", dg.T @ X)
    return dg @ W["gen.in"]


def shard_rows(n: int, P: int, r: int):
    return (r * n) // P, ((r + 1) * n) // P


# ----------------------------------------------------------------------------
# the plain reference: sequential microbatches, full fwd then full bwd
# ----------------------------------------------------------------------------
def to_f64(weights):
    return {k: np.asarray(v, dtype=np.float64) for k, v in weights.items()}


def microbatch_fwd_bwd(W, cfg, batch, m, G, scale):
    """Loss terms (ce, mse) of microbatch m; accumulates scale * grad into G."""
    n_mod = int(batch.n_mod[m])
    n_gen = int(batch.n_gen[m])
    patches = np.asarray(batch.patches[m], np.float64)
    ids, labels = batch.ids[m], batch.labels[m]
    t = np.asarray(batch.targets[m], np.float64)
    S = cfg.S

    E, ecache = encoder_fwd(W, cfg, patches)
    X = embed_fwd(W, ids, E, n_mod)
    H, lcache = llm_layers_fwd(W, cfg, list(range(cfg.L)), X)
    Hn, ce, hcache = head_fwd(W, cfg, H, labels, n_mod)
    denom = float(n_gen * cfg.d_t)
    mse, gcache = gen_fwd(W, cfg, Hn[S - n_gen:], t, denom)

    dXg = gen_bwd(W, cfg, gcache, scale, G)
    dHn = head_bwd_logits(W, cfg, hcache, scale, G)
    dHn[S - n_gen:] += dXg
    dH = final_norm_bwd(W, hcache, dHn, G)
    dX = llm_layers_bwd(W, cfg, list(range(cfg.L)), lcache, dH, G)
    dE = embed_bwd(cfg, dX, ids, n_mod, G)
    encoder_bwd(W, cfg, ecache, dE, G)
    return ce, mse


def step_fp64(cfg, weights, batch):
    """Returns (loss, per-mb [(ce, mse)], grads) for L = (1/M) sum_m (CE_m + MSE_m)."""
    W = to_f64(weights)
    M = len(batch.n_mod)
    G = {}
    per_mb = []
    for m in range(M):
        per_mb.append(microbatch_fwd_bwd(W, cfg, batch, m, G, 1.0 / M))
    loss = sum(ce + mse for ce, mse in per_mb) / M
    for k in W:
        if k not in G:
            G[k] = np.zeros_like(W[k])
    return loss, per_mb, G


def loss_only(cfg, weights, batch):
    """Forward-only loss, used by the finite-difference pin."""
    W = to_f64(weights)
    M = len(batch.n_mod)
    tot = 0.0
    for m in range(M):
        n_mod, n_gen = int(batch.n_mod[m]), int(batch.n_gen[m])
        E, _ = encoder_fwd(W, cfg, np.asarray(batch.patches[m], np.float64))
        X = embed_fwd(W, batch.ids[m], E, n_mod)
        H, _ = llm_layers_fwd(W, cfg, list(range(cfg.L)), X)
        Hn, ce, _ = head_fwd(W, cfg, H, batch.labels[m], n_mod)
        mse, _ = gen_fwd(W, cfg, Hn[cfg.S - n_gen:], np.asarray(batch.targets[m], np.float64),
                         float(n_gen * cfg.d_t))
        tot += ce + mse
    return tot / M
