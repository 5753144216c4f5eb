"""GPU parity of the device Matern kernel and the dense fp64 check path against
the oracle (Eq. 1 and Eq. 2).  Tolerance: 1e-10 relative on the
log-likelihood (north star), 1e-12 relative on kernel entries."""
import math

import numpy as np
import pytest

from oracle import dense as odense
from oracle.matern import matern as omatern
from synthetic import uniform_iid, standard_normal, perturbed_mesh

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def hm(gpu_required):
    import paper_1709_04419_b200 as hm
    return hm


@pytest.mark.parametrize("nu", [0.5, 1.5, 2.5, 1.0, 0.35, 0.73, 3.2, 0.1, 5.6])
def test_matern_kernel_vs_oracle(hm, nu):
    rng = np.random.default_rng(17)
    a = rng.random((64, 2))
    b = rng.random((50, 2)) * 3.0
    theta = (1.7, 0.13, nu)
    got = hm.matern_block(a, b, theta)
    h = np.sqrt(((a[:, None, :] - b[None, :, :]) ** 2).sum(-1))
    want = omatern(h.ravel(), *theta).reshape(h.shape)
    np.testing.assert_allclose(got, want, rtol=1e-12, atol=1e-300)
    # zero lag and tiny lags (continuity)
    z = hm.matern_block(np.array([[0.2, 0.2]]), np.array([[0.2, 0.2], [0.2, 0.2 + 1e-9]]), theta)
    assert z[0, 0] == 1.7
    h_tiny = (0.2 + 1e-9) - 0.2          # the lag the kernel actually sees (not exactly 1e-9)
    assert z[0, 1] == pytest.approx(omatern(h_tiny, *theta)[0], rel=1e-12)


def _check_dense(hm, pts, theta, Z, rtol=1e-10):
    """North star: 1e-10 relative.  For an ill-conditioned C and a Z that is not
    drawn from the model, two correct fp64 Cholesky solves (the oracle in two
    point orders) already differ by more than that (kappa(C) * u); the bar is then
    10x that measured rounding floor ('tolerances')."""
    got = hm.dense_loglik(pts, theta, Z)
    bessel = "quad" if len(pts) <= 2500 else "scipy"
    C = odense.covariance(pts, theta, bessel=bessel)
    ll, ld, q = odense.loglik_from_cov(C, Z)
    p = np.random.default_rng(0).permutation(len(pts))
    ll2, ld2, q2 = odense.loglik_from_cov(C[np.ix_(p, p)], np.asarray(Z)[p])
    ll, q, ll2, q2 = (np.atleast_1d(v) for v in (ll, q, ll2, q2))
    floor = lambda a, b: float(np.max(np.abs(a - b) / np.abs(a)))
    np.testing.assert_allclose(got[:, 0], ll, rtol=max(rtol, 10 * floor(ll, ll2)))
    np.testing.assert_allclose(got[:, 1], ld, rtol=max(rtol, 10 * abs(ld - ld2) / abs(ld)), atol=rtol * len(pts))
    np.testing.assert_allclose(got[:, 2], q, rtol=max(rtol, 10 * floor(q, q2)))


def test_dense_config0(hm):
    # configs[0]: n = 2000 uniform, sigma^2 = 1, ell = 0.0864, nu = 0.5, Z = L N(0, I)
    pts = uniform_iid(2000, seed=0)
    theta = (1.0, 0.0864, 0.5)
    Z = odense.sample(pts, theta, standard_normal(2000, 1, seed=1))
    _check_dense(hm, pts, theta, Z)


@pytest.mark.parametrize("n,nu,k", [(777, 1.0, 1), (1, 0.5, 1), (63, 1.5, 3), (65, 0.35, 2), (1500, 2.2, 70)])
def test_dense_ragged_general_nu(hm, n, nu, k):
    pts = uniform_iid(n, seed=n)
    theta = (1.3, 0.11, nu)
    Z = standard_normal(n, k, seed=2)
    _check_dense(hm, pts, theta, Z)


def test_dense_16k(hm):
    # configs[1]: n = 16384 uniform, theta = (1, 0.2, 1.5), Z = L xi from the dense
    # Cholesky of the true C (model-drawn data, as configs[0] states)
    pts = uniform_iid(16384, seed=1)
    theta = (1.0, 0.2, 1.5)
    C = odense.covariance(pts, theta, bessel="scipy")
    L = np.linalg.cholesky(C)
    Z = L @ standard_normal(16384, 1, seed=3)
    got = hm.dense_loglik(pts, theta, Z)
    ll, ld, q = odense.loglik_from_cov(C, Z)
    assert abs(got[0, 0] - ll) <= 1e-10 * abs(ll)
    assert abs(got[0, 1] - ld) <= 1e-10 * abs(ld)


def test_dense_device_pointers(hm):
    import torch
    pts = uniform_iid(500, seed=5)
    Z = standard_normal(500, 2, seed=6)
    theta = (1.0, 0.1, 0.8)
    host = hm.dense_loglik(pts, theta, Z)
    dev = hm.dense_loglik(torch.tensor(pts, device="cuda"), theta, torch.tensor(Z.T.copy(), device="cuda"))
    np.testing.assert_allclose(dev, host, rtol=1e-13)


def test_dense_errors(hm):
    with pytest.raises(hm.HMError):
        hm.dense_loglik(uniform_iid(10, 0), (1.0, -0.1, 0.5), np.zeros(10))
    with pytest.raises(hm.HMError) as e:
        hm.dense_loglik(uniform_iid(131073, 0), (1.0, 0.1, 0.5), np.zeros(131073))
    assert e.value.code == -7
    with pytest.raises(ValueError):
        hm.dense_loglik(uniform_iid(10, 0), (1.0, 0.1, 0.5), np.zeros(11))


def test_dense_65536_exponential_line_closed_form(hm):
    """The dense check path at configs[2]'s size (n = 65,536, the reference of the
    full-size mesh tests): exponential covariance on an equispaced line has
    log det C = n log sigma^2 + (n-1) log(1 - rho^2) and a tridiagonal inverse
    (the closed forms pinned in test_oracle_dense.py), Z drawn by the AR(1)
    recursion.  North-star bar 1e-10 relative."""
    import math
    n, sigma2, ell = 65536, 1.3, 0.1
    pts = np.stack([(np.arange(n) + 0.5) / n, np.zeros(n)], axis=1)
    rho = math.exp(-1.0 / (n * ell))
    xi = standard_normal(n, 1, seed=40)[:, 0]
    z = np.empty(n)
    z[0] = math.sqrt(sigma2) * xi[0]
    s = math.sqrt(sigma2 * (1 - rho * rho))
    for i in range(1, n):
        z[i] = rho * z[i - 1] + s * xi[i]
    logdet = n * math.log(sigma2) + (n - 1) * math.log1p(-rho * rho)
    quad = ((1 + rho * rho) * np.sum(z * z) - rho * rho * (z[0] ** 2 + z[-1] ** 2)
            - 2 * rho * np.sum(z[:-1] * z[1:])) / (sigma2 * (1 - rho * rho))
    ll = -0.5 * n * math.log(2 * math.pi) - 0.5 * logdet - 0.5 * quad
    got = hm.dense_loglik(pts, (sigma2, ell, 0.5), z)[0]
    assert abs(got[0] - ll) <= 1e-10 * abs(ll)
    assert abs(got[1] - logdet) <= 1e-10 * abs(logdet)
    assert abs(got[2] - quad) <= 1e-10 * abs(ll)
