"""Oracle: Matern covariance, sec. 2.2, Eq. (2) (l.183-188).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

    C(h; theta) = sigma^2 / (2^(nu-1) Gamma(nu)) * (h/ell)^nu * K_nu(h/ell),
    theta = (sigma^2, ell, nu)                                       (Eq. 2)

taken literally (no sqrt(2 nu) inside h/ell -- DESIGN.md reading R5), with
C(0) = sigma^2 (the h -> 0 limit, since x^nu K_nu(x) -> 2^(nu-1) Gamma(nu)).

K_nu ("the modified Bessel function of the second kind of order nu", l.188)
is evaluated from its integral representation

    K_nu(x) = int_0^inf exp(-x cosh t) cosh(nu t) dt        (x > 0)

by the trapezoidal rule with step H = 1/16 on [0, T(x)].  The integrand is analytic
in the strip |Im t| < pi/2 and decays double-exponentially, so the rule's
error is O(exp(-pi^2 / H)) for moderate x (O(exp(-2 pi^2/(H^2 x))) for large x);
H = 1/16 leaves it below 1e-16 relative for x <= 100, and
T is taken where x cosh T - nu T exceeds the largest log-term by 60.
``bessel="scipy"`` swaps in scipy.special.kv (a library routine, used only to
reach larger n quickly; both are pinned against each other in tests).
"""
from __future__ import annotations

import math

import numpy as np

_H = 1.0 / 16.0


def bessel_k(nu: float, x) -> np.ndarray:
    """K_nu(x) for x > 0 (vectorised over x) by trapezoidal quadrature."""
    x = np.atleast_1d(np.asarray(x, dtype=np.float64))
    if np.any(~(x > 0)):
        raise ValueError("bessel_k: x > 0 required")
    nu = abs(float(nu))                      # K_{-nu} = K_nu
    xmin = float(x.min())
    # exponent g(t) = -x cosh t + nu t peaks at t* = asinh(nu/x) with value
    # g* = nu asinh(nu/x) - sqrt(x^2 + nu^2); subtract it per element so exp()
    # stays in range for tiny x / large nu, and stop at T where the smallest x
    # has fallen 60 below its peak (e^-60 ~ 1e-26 relative tail).
    scale = nu * np.arcsinh(nu / x) - np.sqrt(x * x + nu * nu)
    gmin = nu * math.asinh(nu / xmin) - math.sqrt(xmin * xmin + nu * nu)
    T = max(1.0, math.asinh(nu / xmin))          # start at the smallest x's peak
    while -xmin * math.cosh(T) + nu * T > gmin - 60.0:
        T += 0.25
    nodes = np.arange(0.0, T + _H, _H)
    acc = np.zeros_like(x)
    for k, t in enumerate(nodes):
        w = 0.5 if k == 0 else 1.0
        acc += w * np.exp(-x * math.cosh(t) + nu * t - scale) * (0.5 * (1.0 + math.exp(-2.0 * nu * t)))
    return acc * _H * np.exp(scale)


def bessel_k_scipy(nu: float, x) -> np.ndarray:
    from scipy.special import kv
    return kv(float(nu), np.asarray(x, dtype=np.float64))


def matern(h, sigma2: float, ell: float, nu: float, bessel: str = "quad") -> np.ndarray:
    """Eq. (2) for distances h >= 0 (vectorised)."""
    h = np.atleast_1d(np.asarray(h, dtype=np.float64))
    if np.any(h < 0) or not np.all(np.isfinite(h)):
        raise ValueError("matern: finite h >= 0 required")
    if not (sigma2 > 0 and ell > 0 and nu > 0):
        raise ValueError("matern: sigma2, ell, nu > 0 required")
    out = np.full(h.shape, float(sigma2))
    pos = h > 0
    if np.any(pos):
        x = h[pos] / ell
        kfun = bessel_k if bessel == "quad" else bessel_k_scipy
        k = kfun(nu, x)
        coef = sigma2 / (2.0 ** (nu - 1.0) * math.gamma(nu))
        out[pos] = coef * np.power(x, nu) * k
    return out
