"""Frozen workload configurations C1..C5 (BASELINE.json `configs[0..4]`).

Shapes marked ‡ in SURVEY.md §8 are proposals; they are frozen here and in
DESIGN.md §"Input recipe".  The synthetic model is an
encoder -> projector -> LLM -> generator of token-wise residual MLP blocks
(SURVEY.md §8(c) Q11): no attention, so per-mb LLM cost depends only on S and
encoder/generator cost only on the per-sample modality row counts.
"""
from __future__ import annotations

import dataclasses
from dataclasses import dataclass, field


@dataclass(frozen=True)
class ModelShape:
    name: str
    # pipeline (paper's P = pp_size, M = microbatch_num, V = vpp size)
    P: int
    M: int
    V: int
    # LLM sequence length (paper: 8K)
    S: int
    # encoder: patch dim, width, mlp width, depth  (GELU residual blocks)
    d_in: int
    d_e: int
    f_e: int
    L_e: int
    # LLM: width (= projector output), SwiGLU width, depth, vocab
    d: int
    f: int
    L: int
    vocab: int
    # generator: width, mlp width, depth, target dim
    d_g: int
    f_g: int
    L_g: int
    d_t: int
    # per-sample modality / generation row-count laws
    n_mod_law: tuple = ("uniform", 16, 64)
    n_gen_law: tuple = ("uniform", 16, 64)
    llm_sched: str = "1f1b"          # "1f1b" (V == 1) or "interleaved" (V >= 2)
    data_seed: int = 0
    weight_seed: int = 1

    def replace(self, **kw) -> "ModelShape":
        return dataclasses.replace(self, **kw)

    @property
    def layers_per_vstage(self) -> int:
        return self.L // (self.P * self.V)


_C1 = ModelShape(
    name="C1", P=2, M=4, V=1, S=128,
    d_in=48, d_e=64, f_e=256, L_e=2,
    d=128, f=384, L=4, vocab=256,
    d_g=64, f_g=256, L_g=2, d_t=16,
    n_mod_law=("uniform", 16, 64), n_gen_law=("uniform", 16, 64),
)

# parity-medium: C1's structure at sizes that span several GEMM tiles in every
# dimension with ragged tails (row counts not multiples of 128), oracle in seconds
_C1M = ModelShape(
    name="C1M", P=2, M=4, V=1, S=384,
    d_in=200, d_e=128, f_e=384, L_e=2,
    d=256, f=640, L=4, vocab=1000,
    d_g=128, f_g=256, L_g=2, d_t=16,
    n_mod_law=("uniform", 60, 200), n_gen_law=("uniform", 60, 200),
)

# ViT-S-shaped encoder + 1B-shaped LLM + small generator (‡ frozen)
_C2 = ModelShape(
    name="C2", P=4, M=16, V=1, S=4096,
    d_in=588, d_e=384, f_e=1536, L_e=12,
    d=2048, f=8192, L=16, vocab=32000,
    d_g=512, f_g=2048, L_g=4, d_t=16,
    n_mod_law=("loguniform", 256, 1024), n_gen_law=("loguniform", 256, 1024),
)

_C3 = _C2.replace(name="C3", M=32, V=2, llm_sched="interleaved")

# ViT-L-shaped encoder + 7B-shaped LLM + diffusion-head-shaped generator (‡ frozen)
_C4 = ModelShape(
    name="C4", P=8, M=64, V=1, S=8192,
    d_in=588, d_e=1024, f_e=4096, L_e=24,
    d=4096, f=11008, L=32, vocab=32000,
    d_g=1024, f_g=4096, L_g=6, d_t=16,
    n_mod_law=("loguniform", 256, 4096), n_gen_law=("loguniform", 256, 4096),
)

_C5 = _C4.replace(name="C5")   # global-batch sweep M in {8,...,256} at P=8

CONFIGS = {c.name: c for c in (_C1, _C1M, _C2, _C3, _C4, _C5)}


def get_config(name: str, **overrides) -> ModelShape:
    cfg = CONFIGS[name]
    if overrides:
        cfg = cfg.replace(**overrides)
    if cfg.V == 1 and cfg.llm_sched not in ("1f1b", "zb_h1"):
        cfg = cfg.replace(llm_sched="1f1b")
    if cfg.V >= 2 and cfg.llm_sched != "interleaved":
        cfg = cfg.replace(llm_sched="interleaved")
    return cfg
