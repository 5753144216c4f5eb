"""CPU checks of the committed configs[1] goldens (tests/golden/gen_config1.py calls only
oracle/ and synthetic/): the file is self-consistent with the mathematics, independent of
any GPU result.  At theta* the data were drawn as Z = L* xi with L* = chol(C(theta*)), so
Z^T C^-1 Z = ||xi||^2 exactly (up to rounding), and every record satisfies Eq. (1)
L = -n/2 log 2 pi - 1/2 logdet - 1/2 quad."""
import json
import math
import os

import numpy as np

from synthetic import standard_normal, theta_grid_ell_nu

HERE = os.path.dirname(os.path.abspath(__file__))
G = json.load(open(os.path.join(HERE, "golden", "config1_oracle.json")))


def test_theta_star_quadratic_form_is_xi_norm():
    xi = standard_normal(G["n"], 1, seed=3)[:, 0]
    star = G["records"][0]
    assert tuple(star["theta"]) == (1.0, 0.2, 1.5)
    assert abs(star["quad"] - float(xi @ xi)) <= 1e-8 * float(xi @ xi)


def test_records_satisfy_eq1_and_cover_the_grid():
    n = G["n"]
    grid = {tuple(map(float, g)) for g in theta_grid_ell_nu()}
    nus = set()
    for r in G["records"]:
        ll = -0.5 * n * math.log(2 * math.pi) - 0.5 * r["logdet"] - 0.5 * r["quad"]
        assert abs(ll - r["loglik"]) <= 1e-12 * abs(r["loglik"]) + 1e-9
        assert tuple(r["theta"]) in grid or tuple(r["theta"]) == (1.0, 0.2, 1.5)
        nus.add(r["theta"][2])
    assert len(G["records"]) == 26 and min(nus) == 0.3 and max(nus) == 2.0
    assert G["records"][0]["lambda_min"] > 0.0


def test_golden_z_is_from_the_generator_seed():
    Z = np.load(os.path.join(HERE, "golden", "config1_Z.npy"))
    assert Z.shape == (G["n"],) and np.all(np.isfinite(Z))
