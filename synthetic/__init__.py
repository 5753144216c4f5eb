"""Seeded synthetic inputs shared by the oracle-side tests and the CUDA path.

This module holds NO arithmetic of the method (no covariance, no Bessel, no
factorisation): only location sets, standard-normal draws and parameter
schedules, all seeded with numpy's PCG64 so both sides see identical bytes.

Workload recipes (PAPER.md line / BASELINE.json config they stand in for):

* ``uniform_iid(n, seed)``          -- configs[0], [1], [3]: n points iid U([0,1]^2).
* ``perturbed_mesh(sqrt_n, delta, seed)`` -- PAPER.md l.203-208, Eq. (3)
  ``((i-0.5+X_ij)/sqrt(n), (j-0.5+Y_ij)/sqrt(n))`` with X, Y iid U(-delta, delta),
  ordered lexicographically by (i, j); configs[2] is sqrt_n=256, delta=0.4.
* ``latlon_dropout(n, seed)``       -- configs[4]: a 0.0067 deg grid over a
  15 x 10 deg box, 30 % seeded dropout, iid jitter U(-0.4h, 0.4h), then a seeded
  subsample of exactly n points (stand-in for the soil-moisture locations of
  PAPER.md l.389, which are not available).
* ``standard_normal(n, k, seed)``   -- xi ~ N(0, I) columns.
"""
from __future__ import annotations

import numpy as np

__all__ = [
    "uniform_iid",
    "perturbed_mesh",
    "latlon_dropout",
    "standard_normal",
    "theta_grid_ell_nu",
]


def _rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(int(seed)))


def uniform_iid(n: int, seed: int) -> np.ndarray:
    """n x 2 float64 locations iid uniform on [0,1]^2."""
    if n < 1:
        raise ValueError("n >= 1 required")
    return _rng(seed).random((n, 2), dtype=np.float64)


def perturbed_mesh(sqrt_n: int, delta: float, seed: int) -> np.ndarray:
    """PAPER.md Eq. (3) (l.203-208): jittered sqrt_n x sqrt_n lattice in [0,1]^2.

    Row k = (i-1)*sqrt_n + (j-1) holds the point for the pair (i, j), i.e. the
    lexicographic order the paper states.
    """
    if sqrt_n < 1:
        raise ValueError("sqrt_n >= 1 required")
    if not (0.0 <= delta < 0.5):
        raise ValueError("perturbation must satisfy 0 <= delta < 0.5")
    rng = _rng(seed)
    m = sqrt_n
    n = m * m
    jit = rng.uniform(-delta, delta, size=(n, 2)) if delta > 0 else np.zeros((n, 2))
    i = np.repeat(np.arange(1, m + 1, dtype=np.float64), m)
    j = np.tile(np.arange(1, m + 1, dtype=np.float64), m)
    pts = np.empty((n, 2), dtype=np.float64)
    pts[:, 0] = (i - 0.5 + jit[:, 0]) / m
    pts[:, 1] = (j - 0.5 + jit[:, 1]) / m
    return pts


def latlon_dropout(n: int, seed: int, h: float = 0.0067,
                   box=(15.0, 10.0), keep: float = 0.7) -> np.ndarray:
    """configs[4] stand-in: jittered lat/lon grid with seeded dropout.

    Grid nodes ((i+0.5)h, (j+0.5)h) inside a box[0] x box[1] degree box, each
    kept with probability ``keep``, jittered by iid U(-0.4h, 0.4h) per axis,
    then exactly n of the survivors drawn without replacement (sorted back into
    grid order).
    """
    rng = _rng(seed)
    nx = int(np.floor(box[0] / h))
    ny = int(np.floor(box[1] / h))
    mask = rng.random(nx * ny) < keep
    idx = np.nonzero(mask)[0]
    if idx.size < n:
        raise ValueError(f"only {idx.size} grid nodes survive dropout, need {n}")
    pick = np.sort(rng.choice(idx, size=n, replace=False))
    gi = (pick // ny).astype(np.float64)
    gj = (pick % ny).astype(np.float64)
    jit = rng.uniform(-0.4 * h, 0.4 * h, size=(n, 2))
    pts = np.empty((n, 2), dtype=np.float64)
    pts[:, 0] = (gi + 0.5) * h + jit[:, 0]
    pts[:, 1] = (gj + 0.5) * h + jit[:, 1]
    return pts


def standard_normal(n: int, k: int, seed: int) -> np.ndarray:
    """n x k iid N(0,1) float64 (column-major friendly: returned C-contiguous n x k)."""
    out = _rng(seed).standard_normal((n, k))
    return np.ascontiguousarray(out)


def theta_grid_ell_nu(sigma2: float = 1.0, n_ell: int = 20, n_nu: int = 20,
                      ell_range=(0.05, 0.4), nu_range=(0.3, 2.0)) -> np.ndarray:
    """configs[1]: a 20 x 20 (ell, nu) grid at fixed sigma^2 (ranges are our reading,
    DESIGN.md 'readings'); returns (n_ell*n_nu) x 3 rows (sigma2, ell, nu)."""
    ells = np.geomspace(ell_range[0], ell_range[1], n_ell)
    nus = np.linspace(nu_range[0], nu_range[1], n_nu)
    g = np.array([(sigma2, e, v) for e in ells for v in nus], dtype=np.float64)
    return g
