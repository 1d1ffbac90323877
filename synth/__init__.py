"""Seeded synthetic inputs and the BASELINE.json configurations.

Shared by tests/ and bench.py (and the only module both the CUDA path's callers
and the oracle's callers use).  It holds NO arithmetic of the method: only the
random-number recipe and the configuration table.
"""

import numpy as np

# BASELINE.json "configs" (d, p, n_el per direction).  n_s = n_el + p - 2,
# n_t = n_el + p - 1 (reading c1).
CONFIGS = {
    1: {"d": 1, "p": 2, "n_el": 16, "what": "2D space-time square; dense-P check"},
    2: {"d": 2, "p": 3, "n_el": 64, "what": "3D space-time cube; fd throughput + PCG (kind 0)"},
    3: {"d": 3, "p": 3, "n_el": 64, "what": "4D hypercube; single-GPU roofline case"},
    4: {"d": 3, "p": 6, "n_el": 128, "what": "4D hypercube; 1/2/4/8-GPU slab-partitioned fd_apply"},
    5: {"d": 3, "p": (2, 4, 8), "n_el": 96, "what": "PCG robustness in p (kind 1)"},
}


def residual(shape, seed):
    """r ~ U[-1, 1] fp64 from numpy default_rng(seed): generated
    globally in colex order, so every rank / GPU count sees the same tensor."""
    return np.random.default_rng(seed).uniform(-1.0, 1.0, size=shape)


def rank1_factors(lengths, seed):
    """Independent U[-1,1] vectors (slowest axis first) for rank-1 inputs whose
    exact FD image can be sampled entry by entry at full size."""
    rng = np.random.default_rng(seed)
    return [rng.uniform(-1.0, 1.0, size=n) for n in lengths]


def rank1_tensor(factors):
    out = factors[0]
    for v in factors[1:]:
        out = np.multiply.outer(out, v)
    return out
