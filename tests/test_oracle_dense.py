"""Pins for oracle.dense (Eq. 1, l.52-55; l.265; l.283).

Each pin is independent of the oracle's own arithmetic path (LAPACK Cholesky):
  * the exponential covariance on a regular 1-D grid (an AR(1) Toeplitz matrix)
    has det = sigma^(2n) (1 - rho^2)^(n-1), rho = e^{-h/ell}, and a tridiagonal
    inverse  (sigma^2 (1-rho^2))^{-1} tridiag(-rho; 1, 1+rho^2, ..., 1+rho^2, 1; -rho);
  * brute force for n <= 7: Leibniz determinant and adjugate inverse;
  * the SPEC hand cases (2x2 [[4,2],[2,3]], n = 1, C = I).
"""
import itertools
import math

import numpy as np
import pytest

from oracle import dense
from synthetic import uniform_iid, standard_normal

LOG2PI = math.log(2 * math.pi)


def leibniz_det(a):
    n = a.shape[0]
    tot = 0.0
    for p in itertools.permutations(range(n)):
        inv = sum(1 for i in range(n) for j in range(i + 1, n) if p[i] > p[j])
        prod = 1.0
        for i in range(n):
            prod *= a[i, p[i]]
        tot += -prod if inv % 2 else prod
    return tot


def adjugate_inverse(a):
    n = a.shape[0]
    d = leibniz_det(a)
    inv = np.empty_like(a)
    for i in range(n):
        for j in range(n):
            minor = np.delete(np.delete(a, j, axis=0), i, axis=1)
            inv[i, j] = (-1) ** (i + j) * leibniz_det(minor) / d
    return d, inv


@pytest.mark.parametrize("n,h,ell,sigma2", [(40, 0.05, 0.1, 1.0), (250, 0.01, 0.0864, 2.0), (7, 0.3, 0.2, 0.5)])
def test_exponential_1d_grid_closed_forms(n, h, ell, sigma2):
    pts = np.zeros((n, 2))
    pts[:, 0] = np.arange(n) * h
    z = standard_normal(n, 1, seed=11)[:, 0]
    ll, logdet, quad = dense.loglik(pts, z, (sigma2, ell, 0.5))
    rho = math.exp(-h / ell)
    logdet_exact = n * math.log(sigma2) + (n - 1) * math.log(1 - rho * rho)
    assert logdet == pytest.approx(logdet_exact, rel=1e-11, abs=1e-10)
    diag = np.full(n, 1 + rho * rho)
    diag[0] = diag[-1] = 1.0
    quad_exact = (np.sum(diag * z * z) - 2 * rho * np.sum(z[:-1] * z[1:])) / (sigma2 * (1 - rho * rho))
    assert quad == pytest.approx(quad_exact, rel=1e-10)
    assert ll == pytest.approx(-0.5 * n * LOG2PI - 0.5 * logdet_exact - 0.5 * quad_exact, rel=1e-11)


@pytest.mark.parametrize("n,nu", [(2, 0.5), (5, 1.5), (6, 0.8), (7, 2.3)])
def test_brute_force_small(n, nu):
    pts = uniform_iid(n, seed=100 + n)
    theta = (1.3, 0.25, nu)
    C = dense.covariance(pts, theta)
    z = standard_normal(n, 1, seed=7)[:, 0]
    d, inv = adjugate_inverse(C)
    ll, logdet, quad = dense.loglik(pts, z, theta)
    assert logdet == pytest.approx(math.log(d), rel=1e-9, abs=1e-10)
    assert quad == pytest.approx(float(z @ inv @ z), rel=1e-9)
    assert ll == pytest.approx(-0.5 * n * LOG2PI - 0.5 * math.log(d) - 0.5 * float(z @ inv @ z), rel=1e-10)


def test_hand_2x2():
    C = np.array([[4.0, 2.0], [2.0, 3.0]])
    ll, logdet, quad = dense.loglik_from_cov(C, np.array([1.0, 1.0]))
    assert logdet == pytest.approx(math.log(8.0), rel=1e-15)
    assert quad == pytest.approx(3.0 / 8.0, rel=1e-15)
    assert ll == pytest.approx(-LOG2PI - 0.5 * math.log(8.0) - 3.0 / 16.0, rel=1e-15)


def test_n1_and_identity():
    ll, logdet, quad = dense.loglik(np.array([[0.3, 0.4]]), np.array([0.0]), (1.0, 0.1, 0.5))
    assert ll == pytest.approx(-0.5 * LOG2PI)
    assert logdet == 0.0 and quad == 0.0
    far = np.array([[0.0, 0.0], [1e3, 0.0]])          # C = I to machine precision
    ll, logdet, quad = dense.loglik(far, np.array([1.0, 1.0]), (1.0, 0.01, 0.5))
    assert ll == pytest.approx(-LOG2PI - 1.0, rel=1e-15)


def test_covariance_symmetric_and_diag():
    pts = uniform_iid(60, seed=3)
    C = dense.covariance(pts, (2.0, 0.1, 0.9))
    assert np.array_equal(C, C.T)
    assert np.all(np.diag(C) == 2.0)
    assert np.all(np.linalg.eigvalsh(C) > 0)


def test_permutation_invariance_and_multicolumn():
    pts = uniform_iid(120, seed=5)
    theta = (1.0, 0.0864, 0.5)
    z = standard_normal(120, 3, seed=9)
    ll, logdet, quad = dense.loglik(pts, z, theta)
    perm = np.random.default_rng(2).permutation(120)
    ll2, logdet2, quad2 = dense.loglik(pts[perm], z[perm], theta)
    np.testing.assert_allclose(ll, ll2, rtol=1e-10)
    assert logdet == pytest.approx(logdet2, rel=1e-10, abs=1e-9)
    for k in range(3):
        llk, _, qk = dense.loglik(pts, z[:, k], theta)
        assert llk == pytest.approx(ll[k], rel=1e-12)
        assert qk == pytest.approx(quad[k], rel=1e-12)


def test_sample_covariance_structure():
    # Z = L xi reproduces C in expectation: E[Z Z^T] = L L^T = C
    pts = uniform_iid(5, seed=21)
    theta = (1.0, 0.3, 1.5)
    xi = standard_normal(5, 40000, seed=4)
    Z = dense.sample(pts, theta, xi)
    emp = Z @ Z.T / xi.shape[1]
    np.testing.assert_allclose(emp, dense.covariance(pts, theta), atol=4 / math.sqrt(40000) * 2)
