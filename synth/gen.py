"""Counter-seeded synthetic data and weights.

Recipe (also stated in DESIGN.md):
  * n_mod, n_gen per sample: C1 uniform integers in [16, 64]; C2/C3
    log-uniform in [256, 1024]; C4/C5 log-uniform in [256, 4096]; independent
    draws, data seed 0 (PCG64).
  * patches ~ N(0, 1); ids, labels ~ U[0, vocab); targets ~ N(0, 1).
  * weights ~ N(0, 0.02); residual-branch output projections (encoder fc2,
    LLM down, generator fc2) scaled by 1/sqrt(2 L_module); RMSNorm gains = 1.
    Each tensor has its own SeedSequence([weight_seed, crc32(name)]) so any
    rank can materialise only the tensors it owns.
  * every floating value is rounded to the nearest bf16 (round-to-nearest-
    even) and returned as float32, so the oracle (fp64) and the CUDA path
    (bf16 or fp32) start from bit-identical inputs.
No arithmetic of the method lives here.
"""
from __future__ import annotations

import zlib
from dataclasses import dataclass

import numpy as np

from .configs import ModelShape


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round to the nearest bf16 value (ties to even); returns float32."""
    a = np.ascontiguousarray(x, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    bias = 0x7FFF + ((u >> 16) & 1)
    r = ((u + bias) & 0xFFFF0000).astype(np.uint32)
    return r.view(np.float32).reshape(a.shape)


# ----------------------------------------------------------------------------
# parameters
# ----------------------------------------------------------------------------
def param_specs(cfg: ModelShape):
    """Logical parameter list: (name, shape, kind) with kind in {"w","wout","g"}.

    Linear weights are stored [out, in] (y = x W^T).  LLM gate_up is [2f, d]
    with rows [0, f) the gate and [f, 2f) the up projection.
    """
    s = []
    s.append(("enc.patch", (cfg.d_e, cfg.d_in), "w"))
    for i in range(cfg.L_e):
        s.append((f"enc.blk{i}.norm", (cfg.d_e,), "g"))
        s.append((f"enc.blk{i}.fc1", (cfg.f_e, cfg.d_e), "w"))
        s.append((f"enc.blk{i}.fc2", (cfg.d_e, cfg.f_e), "wout_enc"))
    s.append(("enc.proj1", (cfg.d, cfg.d_e), "w"))
    s.append(("enc.proj2", (cfg.d, cfg.d), "w"))
    s.append(("llm.embed", (cfg.vocab, cfg.d), "w"))
    for l in range(cfg.L):
        s.append((f"llm.layer{l}.norm", (cfg.d,), "g"))
        s.append((f"llm.layer{l}.gate_up", (2 * cfg.f, cfg.d), "w"))
        s.append((f"llm.layer{l}.down", (cfg.d, cfg.f), "wout_llm"))
    s.append(("llm.final_norm", (cfg.d,), "g"))
    s.append(("llm.head", (cfg.vocab, cfg.d), "w"))
    s.append(("gen.in", (cfg.d_g, cfg.d), "w"))
    for i in range(cfg.L_g):
        s.append((f"gen.blk{i}.norm", (cfg.d_g,), "g"))
        s.append((f"gen.blk{i}.fc1", (cfg.f_g, cfg.d_g), "w"))
        s.append((f"gen.blk{i}.fc2", (cfg.d_g, cfg.f_g), "wout_gen"))
    s.append(("gen.out", (cfg.d_t, cfg.d_g), "w"))
    return s


def _tensor_rng(seed: int, name: str) -> np.random.Generator:
    ss = np.random.SeedSequence([seed, zlib.crc32(name.encode())])
    return np.random.Generator(np.random.PCG64(ss))


def make_weights(cfg: ModelShape, names=None, std: float = 0.02) -> dict:
    """Return {name: float32 array (bf16-representable)} for `names` (all if None)."""
    out = {}
    want = None if names is None else set(names)
    depth = {"wout_enc": cfg.L_e, "wout_llm": cfg.L, "wout_gen": cfg.L_g}
    for name, shape, kind in param_specs(cfg):
        if want is not None and name not in want:
            continue
        if kind == "g":
            out[name] = np.ones(shape, np.float32)
            continue
        scale = std
        if kind in depth:
            scale = std / np.sqrt(2.0 * depth[kind])
        rng = _tensor_rng(cfg.weight_seed, name)
        w = rng.standard_normal(shape, dtype=np.float32) * np.float32(scale)
        out[name] = bf16_round(w)
    return out


# ----------------------------------------------------------------------------
# data
# ----------------------------------------------------------------------------
@dataclass
class Batch:
    n_mod: np.ndarray          # [M] int64
    n_gen: np.ndarray          # [M] int64
    patches: list              # M x [n_mod[m], d_in] float32
    ids: np.ndarray            # [M, S] int32
    labels: np.ndarray         # [M, S] int32
    targets: list              # M x [n_gen[m], d_t] float32


def _draw_counts(rng, law, M, S):
    kind, lo, hi = law
    if kind == "uniform":
        n = rng.integers(lo, hi + 1, size=M)
    elif kind == "loguniform":
        u = rng.uniform(np.log(lo), np.log(hi + 1), size=M)
        n = np.floor(np.exp(u)).astype(np.int64)
    else:
        raise ValueError(kind)
    return np.clip(n, 1, S).astype(np.int64)


def make_batch(cfg: ModelShape, seed: int | None = None, M: int | None = None, n_mod=None, n_gen=None) -> Batch:
    """Seeded synthetic batch.  n_mod / n_gen: explicit per-microbatch row counts
    (edge cases: 0 modality rows, n_mod = S -- no text rows --, fewer generator rows
    than ranks, modality and generator rows overlapping) instead of the laws."""
    seed = cfg.data_seed if seed is None else seed
    M = cfg.M if M is None else M
    rng = np.random.Generator(np.random.PCG64(seed))
    drawn_mod = _draw_counts(rng, cfg.n_mod_law, M, cfg.S)
    drawn_gen = _draw_counts(rng, cfg.n_gen_law, M, cfg.S)
    n_mod = drawn_mod if n_mod is None else np.asarray(n_mod, np.int64)
    n_gen = drawn_gen if n_gen is None else np.asarray(n_gen, np.int64)
    assert len(n_mod) == M and len(n_gen) == M
    assert all(0 <= x <= cfg.S for x in n_mod) and all(1 <= x <= cfg.S for x in n_gen)
    patches, targets = [], []
    ids = np.empty((M, cfg.S), np.int32)
    labels = np.empty((M, cfg.S), np.int32)
    for m in range(M):
        patches.append(bf16_round(rng.standard_normal((int(n_mod[m]), cfg.d_in), dtype=np.float32)))
        ids[m] = rng.integers(0, cfg.vocab, size=cfg.S)
        labels[m] = rng.integers(0, cfg.vocab, size=cfg.S)
        targets.append(bf16_round(rng.standard_normal((int(n_gen[m]), cfg.d_t), dtype=np.float32)))
    return Batch(n_mod=n_mod, n_gen=n_gen, patches=patches, ids=ids, labels=labels, targets=targets)


def edge_counts(cfg: ModelShape, M: int):
    """The method's degenerate row counts, cycled over M microbatches: no modality
    rows, modality rows filling the sequence (no CE rows), a few modality rows with
    the generator reading the whole sequence (modality, CE and generator rows
    overlap), fewer generator rows than a 4-stage pipeline has ranks (empty
    generator shards).  Returns (n_mod, n_gen)."""
    S = cfg.S
    mods = [0, S, 17, 60]
    gens = [1, 3, S, 2]
    return [mods[m % 4] for m in range(M)], [gens[m % 4] for m in range(M)]


def edge_shape(cfg: ModelShape) -> ModelShape:
    """cfg with row-count laws spanning [0, S] so the buffers admit every edge count."""
    return cfg.replace(n_mod_law=("uniform", 0, cfg.S), n_gen_law=("uniform", 1, cfg.S))


def slice_batch(b: Batch, lo: int, hi: int) -> Batch:
    """Microbatches [lo, hi) of a batch (one pipeline replica's share of a global batch)."""
    return Batch(n_mod=b.n_mod[lo:hi].copy(), n_gen=b.n_gen[lo:hi].copy(), patches=list(b.patches[lo:hi]),
                 ids=b.ids[lo:hi].copy(), labels=b.labels[lo:hi].copy(), targets=list(b.targets[lo:hi]))
