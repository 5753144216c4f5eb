"""Oracle: dense covariance and the exact Gaussian log-likelihood, Eq. (1).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Eq. (1) (l.52-55):
    L(theta) = -n/2 log(2 pi) - 1/2 log det C(theta) - 1/2 Z^T C(theta)^{-1} Z,
with C(theta)_{ij} = C(s_i - s_j; theta) (l.56) and C the Matern kernel (Eq. 2).
Evaluated the way the paper says it is evaluated (sec. 3.1, Eq. 4, l.259-265
and l.283): C = L L^T (library Cholesky, numpy/LAPACK), log det C = 2 sum log L_ii,
v = L^{-1} Z (library triangular solve), Z^T C^{-1} Z = v^T v.
"""
from __future__ import annotations

import math

import numpy as np
import scipy.linalg

from .matern import matern


def covariance(points: np.ndarray, theta, bessel: str = "quad") -> np.ndarray:
    """Dense C(theta) with entries C(s_i - s_j; theta) (l.56).  Each unordered
    pair is evaluated once and mirrored, so the result is exactly symmetric."""
    sigma2, ell, nu = (float(v) for v in theta)
    p = np.asarray(points, dtype=np.float64)
    n = p.shape[0]
    iu, ju = np.triu_indices(n, k=1)
    dx = p[iu, 0] - p[ju, 0]
    dy = p[iu, 1] - p[ju, 1]
    h = np.sqrt(dx * dx + dy * dy)
    c = np.empty((n, n), dtype=np.float64)
    vals = matern(h, sigma2, ell, nu, bessel=bessel) if h.size else h
    c[iu, ju] = vals
    c[ju, iu] = vals
    c[np.arange(n), np.arange(n)] = sigma2
    return c


def loglik_from_cov(C: np.ndarray, Z: np.ndarray):
    """Eq. (1) for a given SPD matrix C and data vector(s) Z (n or n x k).

    Returns (loglik, logdet, quad); for n x k Z, loglik and quad are length-k
    arrays (one replicate per column) and logdet is shared.
    Raises numpy.linalg.LinAlgError if C is not positive definite.
    """
    C = np.asarray(C, dtype=np.float64)
    n = C.shape[0]
    L = np.linalg.cholesky(C)                                   # C = L L^T
    logdet = 2.0 * float(np.sum(np.log(np.diag(L))))            # l.283
    v = scipy.linalg.solve_triangular(L, np.asarray(Z, dtype=np.float64), lower=True)  # L v = Z (l.265)
    quad = np.sum(v * v, axis=0)                                 # v^T v = Z^T C^-1 Z
    ll = -0.5 * n * math.log(2.0 * math.pi) - 0.5 * logdet - 0.5 * quad  # Eq. (1)
    if np.ndim(quad) == 0:
        return float(ll), logdet, float(quad)
    return ll, logdet, quad


def loglik(points: np.ndarray, Z: np.ndarray, theta, bessel: str = "quad"):
    """Eq. (1) at theta = (sigma^2, ell, nu) for locations ``points`` (n x 2) and
    data Z (in the same order as ``points``)."""
    return loglik_from_cov(covariance(points, theta, bessel=bessel), Z)


def sample(points: np.ndarray, theta, xi: np.ndarray, bessel: str = "quad") -> np.ndarray:
    """Z = L xi with C = L L^T (sec. 4, l.308: "Z = L xi"), dense."""
    L = np.linalg.cholesky(covariance(points, theta, bessel=bessel))
    return L @ np.asarray(xi, dtype=np.float64)
