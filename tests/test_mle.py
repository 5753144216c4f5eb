"""Host logic of the MLE driver (paper_1709_04419_b200/mle.py): the Nelder-Mead
search used by configs[3] spends exactly its evaluation budget and converges on
functions with known minimisers."""
import math

import numpy as np
import pytest

from paper_1709_04419_b200.mle import nelder_mead


def test_exact_budget():
    calls = []
    f = lambda x: calls.append(1) or float(np.sum(x * x))
    x, fx, hist = nelder_mead(f, np.array([1.0, 2.0, -1.0]), 0.5, 60)
    assert len(calls) == 60 and len(hist) == 60
    assert fx == min(h[1] for h in hist)


def test_quadratic_minimum():
    c = np.array([0.3, -1.2, 2.0])
    a = np.array([1.0, 10.0, 0.1])
    f = lambda x: float(np.sum(a * (x - c) ** 2))
    x, fx, _ = nelder_mead(f, np.zeros(3), 0.5, 600)
    np.testing.assert_allclose(x, c, atol=1e-3)
    assert fx < 1e-6


def test_rosenbrock():
    f = lambda x: (1 - x[0]) ** 2 + 100 * (x[1] - x[0] ** 2) ** 2
    x, fx, _ = nelder_mead(f, np.array([-1.2, 1.0]), 0.5, 800)
    np.testing.assert_allclose(x, [1.0, 1.0], atol=1e-3)


def test_infinite_values_are_avoided():
    # a region where the objective is undefined (like a failed H-Cholesky) scores +inf
    f = lambda x: math.inf if x[0] > 1.0 else (x[0] - 0.5) ** 2 + x[1] ** 2
    x, fx, _ = nelder_mead(f, np.array([0.9, 0.5]), 0.4, 200)
    assert x[0] <= 1.0 and fx < 1e-4
