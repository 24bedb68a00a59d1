"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This package holds NO arithmetic of the BigMac method: only frozen config
shapes (SURVEY.md §8 header table) and counter-seeded random generators
(SURVEY.md §8(d) "Concrete synthetic inputs", §8(c) Q12).  Both `oracle/`
and `paper_2605_25451_b200/` import it; neither imports the other.
"""
from .configs import CONFIGS, ModelShape, get_config  # noqa: F401
from .gen import (  # noqa: F401
    bf16_round, edge_counts, edge_shape, make_batch, make_weights, param_specs, slice_batch, Batch,
)
