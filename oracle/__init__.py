"""CPU fp64 ORACLE for the H-likelihood hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import or execute anything in this package.
The product path (``paper_1709_04419_b200``) never imports it and shares no code
with it; the two meet only through ``synthetic`` (seeded inputs, no arithmetic).

What it computes, each function citing PAPER.md:

* ``geometry``  -- cluster tree T_I and block cluster tree T_{IxI} (sec. 2.1,
  Definition 1, l.152-160; n_min from l.211) with the readings listed in
  DESIGN.md sec. 3 (median bisection on the longest bounding-box axis,
  admissibility min(diam) <= eta * dist on bounding boxes).
* ``matern``    -- Matern covariance Eq. (2) (l.183-188) with K_nu from its
  integral representation, evaluated by the trapezoidal rule.
* ``dense``     -- C(theta) entries (l.56), dense Cholesky, log det = 2 sum log L_ii
  (l.283), v = L^{-1} Z (l.265), L(theta) of Eq. (1) (l.52-55).

Pins (tests/test_oracle_*.py, ``-m "not gpu"``): closed forms of K_nu and of the
Matern kernel for nu = 1/2, 3/2, 5/2; scipy.special.kv; the Bessel recurrence;
the exact determinant and tridiagonal inverse of the exponential covariance on
a regular 1-D grid; Leibniz/adjugate brute force for n <= 7; hand-built
partitions; exhaustive tiling of I x I.  Parity status of every function is
"pinned"; nothing here is "parity unpinned".
"""
from . import geometry, matern, dense  # noqa: F401
