"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This package holds only input *generation* (random positions, values, filters) and the
COO container types. It contains none of the method's arithmetic (no convolution, no
selection, no pooling), so that the oracle (`oracle/`) and the CUDA path
(`paper_1801_10585_b200/`) share nothing but their inputs.
"""
from .generators import (  # noqa: F401
    COO,
    Filter,
    uniform_map,
    mnist_like,
    surface_occupancy,
    sparse_filter,
    bias_vector,
    grad_values,
    select_samples,
    SEED_BASE,
)
