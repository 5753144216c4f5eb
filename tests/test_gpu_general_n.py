"""General n on the GPU (Def. 1 l.152-160, n_min l.211; Table 1 l.213
allows 1 <= n_min <= 128): trees whose leaves sit at two depths (n / 2^l straddles
n_min) and leaves above one 64 x 64 tile are planned on the refined storage tree
(tree.h refine_for_plan).  The H likelihood must meet the north-star bars against
the dense CPU oracle (small n) or the GPU dense path (n = 16,641 and 65,537, itself
pinned to the oracle / the closed form in test_gpu_dense.py)."""
import numpy as np
import pytest

from oracle import dense as od
from synthetic import perturbed_mesh, standard_normal, uniform_iid

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def hm(gpu_required):
    import paper_1709_04419_b200 as hm
    return hm


def _mixed(hm, pts, leaf):
    t = hm.Tree(pts, leaf, 2.0)
    cl = t.clusters()
    levels = {int(c[2]) for c in cl if c[3]}
    return len(levels) > 1 or max(int(c[1] - c[0]) for c in cl if c[3]) > 64


@pytest.mark.parametrize("n,leaf", [(65, 32), (1040, 32), (777, 48), (1500, 100), (2000, 128), (4128, 64)])
@pytest.mark.parametrize("eps,tol", [(1e-8, 1e-6), (1e-5, 1e-4)])
def test_general_n_vs_oracle(hm, n, leaf, eps, tol):
    pts = uniform_iid(n, seed=100 + n)
    assert _mixed(hm, pts, leaf)
    theta = (1.0, 0.0864, 0.5)
    Z = od.sample(pts, theta, standard_normal(n, 2, seed=7))
    oll, old, oq = od.loglik(pts, Z, theta)
    H = hm.HMatrix(pts, theta, eps=eps, leaf=leaf, eta=2.0)
    H.cholesky()
    got = H.loglik(Z)
    np.testing.assert_allclose(got[:, 0], oll, rtol=tol)


def test_paper_table2_mesh_16641(hm):
    """PAPER.md Table 2 setting (l.228-249): n = 16,641 perturbed mesh (Eq. 3), nu = 0.5,
    sigma^2 = 1, ell in {0.0334, 0.2337}, n_min = 32 -- leaves at two depths."""
    pts = perturbed_mesh(129, 0.4, seed=5)
    assert _mixed(hm, pts, 32)
    for ell in (0.0334, 0.2337):
        theta = (1.0, ell, 0.5)
        Hs = hm.HMatrix(pts, theta, eps=1e-10, leaf=32, eta=2.0)
        Hs.cholesky()
        Z = Hs.sample(standard_normal(len(pts), 1, seed=8))
        Hs.close()
        d = hm.dense_loglik(pts, theta, Z)[0]
        for eps, tol in ((1e-8, 1e-6), (1e-5, 1e-4)):
            H = hm.HMatrix(pts, theta, eps=eps, leaf=32, eta=2.0)
            H.cholesky()
            g = H.loglik(Z)[0]
            assert abs(g[0] - d[0]) <= tol * abs(d[0]), (ell, eps, g, d)
            assert abs(g[1] - d[1]) <= tol * abs(d[0])
            H.close()


def test_65537_leaf64(hm):
    """configs[2]'s size + 1 at leaf 64 (rejected before the storage refinement)."""
    n = 65537
    pts = uniform_iid(n, seed=9)
    assert _mixed(hm, pts, 64)
    theta = (1.0, 0.1, 0.5)
    Hs = hm.HMatrix(pts, theta, eps=1e-10, leaf=64, eta=2.0, kmax=64)
    Hs.cholesky()
    Z = Hs.sample(standard_normal(n, 1, seed=10))
    Hs.close()
    d = hm.dense_loglik(pts, theta, Z)[0]
    H = hm.HMatrix(pts, theta, eps=1e-8, leaf=64, eta=2.0, kmax=64)
    H.cholesky()
    g = H.loglik(Z)[0]
    assert abs(g[0] - d[0]) <= 1e-6 * abs(d[0])
