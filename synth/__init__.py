"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This package holds ONLY input generation: grid geometry, velocity models, source
layouts and random complex fields.  It contains none of the method's arithmetic
(no weights, no coefficients, no operator, no solver), so that `oracle/` and the
CUDA path can both consume it without sharing any method code (task rule ③).

Recipes follow SURVEY.md §8(d) "Synthetic inputs" and BASELINE.json `configs`;
DESIGN.md §"Input recipe" restates them.
"""
from .configs import (  # noqa: F401
    BASE_SEED,
    Config,
    CONFIGS,
    get_config,
    velocity_model,
    velocity_slab,
    crop_config,
    CROP_SHAPE,
    source_nodes,
    random_field,
    rng_for,
)
