"""Pins for oracle.matern (sec. 2.2, Eq. 2, l.183-188).

Independent of the oracle's quadrature: closed forms of K_nu at half-integer
order, scipy.special.kv (library routine), the three-term recurrence, the
x -> 0 limit, and the closed forms of the Matern kernel at nu = 1/2, 3/2, 5/2
(l.188: "When nu = 1/2, the Matern covariance function reduces to the
exponential covariance model").
"""
import math

import numpy as np
import pytest
from scipy.special import kv

from oracle.matern import bessel_k, matern


def k_half(x):      # K_{1/2}(x) = sqrt(pi/(2x)) e^{-x}
    return math.sqrt(math.pi / (2 * x)) * math.exp(-x)


def k_3half(x):     # K_{3/2}(x) = sqrt(pi/(2x)) e^{-x} (1 + 1/x)
    return k_half(x) * (1 + 1 / x)


def k_5half(x):     # K_{5/2}(x) = sqrt(pi/(2x)) e^{-x} (1 + 3/x + 3/x^2)
    return k_half(x) * (1 + 3 / x + 3 / (x * x))


@pytest.mark.parametrize("x", [1e-6, 1e-3, 0.1, 0.7, 1.0, 2.0, 5.0, 17.0, 40.0])
def test_half_integer_closed_forms(x):
    assert bessel_k(0.5, x)[0] == pytest.approx(k_half(x), rel=1e-13)
    assert bessel_k(1.5, x)[0] == pytest.approx(k_3half(x), rel=1e-13)
    assert bessel_k(2.5, x)[0] == pytest.approx(k_5half(x), rel=1e-13)


def test_spec_worked_examples():
    # SPEC.md kernels/bessel_k examples: nu=1/2, x=2 -> sqrt(pi/4) e^-2; nu=3/2, x=1 -> 2 sqrt(pi/2)/e
    assert bessel_k(0.5, 2.0)[0] == pytest.approx(math.sqrt(math.pi / 4) * math.exp(-2), rel=1e-14)
    assert bessel_k(1.5, 1.0)[0] == pytest.approx(2 * math.sqrt(math.pi / 2) / math.e, rel=1e-14)


def test_against_scipy_random():
    rng = np.random.default_rng(20240917)
    nu = rng.uniform(0.1, 5.0, 400)
    x = 10 ** rng.uniform(-4, math.log10(30.0), 400)
    ours = np.array([bessel_k(a, b)[0] for a, b in zip(nu, x)])
    np.testing.assert_allclose(ours, kv(nu, x), rtol=1e-10)


def test_vectorised_matches_scalar():
    x = np.array([1e-5, 0.3, 1.7, 9.0, 33.0])
    vec = bessel_k(0.83, x)
    sca = np.array([bessel_k(0.83, v)[0] for v in x])
    np.testing.assert_allclose(vec, sca, rtol=1e-14)


@pytest.mark.parametrize("nu", [0.35, 1.0, 2.2])
def test_recurrence(nu):
    # K_{nu+1}(x) = K_{nu-1}(x) + (2 nu / x) K_nu(x)  (DLMF 10.29.1)
    for x in [0.05, 0.9, 3.0, 12.0]:
        lhs = bessel_k(nu + 1, x)[0]
        rhs = bessel_k(nu - 1, x)[0] + 2 * nu / x * bessel_k(nu, x)[0]
        assert lhs == pytest.approx(rhs, rel=1e-12)


def test_small_x_limit():
    # x^nu K_nu(x) -> 2^(nu-1) Gamma(nu) as x -> 0 (DLMF 10.30.2)
    for nu in [0.4, 1.3, 2.7]:
        x = 1e-9
        assert x ** nu * bessel_k(nu, x)[0] == pytest.approx(2 ** (nu - 1) * math.gamma(nu), rel=1e-7)


def test_rejects_nonpositive_x():
    with pytest.raises(ValueError):
        bessel_k(0.5, 0.0)


@pytest.mark.parametrize("sigma2,ell", [(1.0, 0.1), (2.5, 0.0864), (0.7, 0.33)])
def test_matern_closed_forms(sigma2, ell):
    h = np.array([1e-7, 0.01, 0.05, 0.1, 0.37, 1.2])
    x = h / ell
    np.testing.assert_allclose(matern(h, sigma2, ell, 0.5), sigma2 * np.exp(-x), rtol=1e-13)
    np.testing.assert_allclose(matern(h, sigma2, ell, 1.5), sigma2 * (1 + x) * np.exp(-x), rtol=1e-13)
    np.testing.assert_allclose(matern(h, sigma2, ell, 2.5),
                               sigma2 * (1 + x + x * x / 3) * np.exp(-x), rtol=1e-13)


def test_matern_zero_lag_and_continuity():
    assert matern(0.0, 1.7, 0.2, 0.8)[0] == 1.7
    # continuity at h -> 0 (SPEC kernels invariant): checked at h = 1e-10 ell
    assert matern(1e-10 * 0.2, 1.7, 0.2, 0.8)[0] == pytest.approx(1.7, rel=1e-7)


def test_matern_monotone_nonincreasing():
    h = np.linspace(0, 2, 400)
    for nu in [0.3, 1.0, 2.3]:
        c = matern(h, 1.0, 0.15, nu)
        assert np.all(np.diff(c) <= 1e-15)


def test_matern_scipy_path_agrees():
    h = np.linspace(1e-4, 1.5, 200)
    np.testing.assert_allclose(matern(h, 1.3, 0.2, 0.73), matern(h, 1.3, 0.2, 0.73, bessel="scipy"),
                               rtol=1e-11)
