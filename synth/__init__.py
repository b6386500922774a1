"""Seeded synthetic inputs shared by the oracle (tests) and the CUDA path.

This package holds NONE of the method's arithmetic: only shape presets
(BASELINE.json:configs) and seeded random-number draws (weights, prompts,
forced-acceptance corruption slots). Both `oracle/` and the product binding
may import it; they share nothing else.
"""
from .configs import ModelConfig, PRESETS, get_config  # noqa: F401
from .weights import weight_shapes, make_weights  # noqa: F401
from .prompts import make_prompts, make_corrupt_slots  # noqa: F401
