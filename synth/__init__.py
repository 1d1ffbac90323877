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


# ---------------------------------------------------------------------------
# Geometry maps F: [0,1]^d -> Omega (PAPER.md 226-250, Ass. 1; Sec. 5 domains).
# Pure data: degree, open knot vector per direction, control points and weights
# (colex order, direction 1 fastest).  Reading c19: the benchmark
# domains are conics, so the map may be rational (NURBS); the discrete space is
# still the push-forward of the B-spline basis (eq:disc_space).
# ---------------------------------------------------------------------------

def _geo(degrees, knots, ctrl, weights):
    return {"d": len(degrees), "degrees": list(degrees),
            "knots": [np.asarray(k, dtype=np.float64) for k in knots],
            "ctrl": np.asarray(ctrl, dtype=np.float64),
            "weights": None if weights is None else np.asarray(weights, dtype=np.float64)}


def affine_box(lengths):
    """x_k = a_k eta_k (degree 1, two control points per direction)."""
    d = len(lengths)
    pts = []
    for idx in np.ndindex(*([2] * d)):
        i = idx[::-1]                                   # colex: direction 1 fastest
        pts.append([lengths[k] * i[k] for k in range(d)])
    return _geo([1] * d, [[0, 0, 1, 1]] * d, pts, None)


_ARC_W = 1.0 / np.sqrt(2.0)        # rational quadratic quarter circle weight


def quarter_annulus():
    """Quarter of the annulus with inner radius 1, outer radius 2 (PAPER.md 1219):
    direction 1 radial (degree 1), direction 2 angular (exact rational quadratic,
    corner control point, weights 1, 1/sqrt 2, 1)."""
    arc = [(1.0, 0.0), (1.0, 1.0), (0.0, 1.0)]
    pts, w = [], []
    for j in range(3):
        for r in (1.0, 2.0):
            pts.append([r * arc[j][0], r * arc[j][1]])
            w.append(1.0 if j != 1 else _ARC_W)
    return _geo([1, 2], [[0, 0, 1, 1], [0, 0, 0, 1, 1, 1]], pts, w)


def revolved_quarter_annulus():
    """That annulus (plane z = 0) revolved by pi/2 about the axis {y = -1, z = 0}
    (PAPER.md 1219, "rotated along the axis y=-1 by pi/2"): direction 3 is the
    revolution angle, each control point revolved by the rational quadratic arc of
    radius rho = y + 1 (corner point construction, weights multiplied)."""
    g2 = quarter_annulus()
    pts, w = [], []
    for j in range(3):
        for c, wc in zip(g2["ctrl"], g2["weights"]):
            x, y = c
            rho = y + 1.0
            q = [(x, y, 0.0), (x, y, rho), (x, -1.0, rho)][j]
            pts.append(q)
            w.append(wc * (1.0 if j != 1 else _ARC_W))
    return _geo([1, 2, 2], [[0, 0, 1, 1], [0, 0, 0, 1, 1, 1], [0, 0, 0, 1, 1, 1]], pts, w)


GEOMETRIES = {"affine": affine_box, "annulus2d": quarter_annulus,
              "annulus3d": revolved_quarter_annulus}
