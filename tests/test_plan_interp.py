"""Host-logic test of the H-Cholesky planner (no GPU): the task DAG that the
GPU executes is interpreted on the CPU (tests/plan_interp.py) with tasks of each
wave in random order, and the resulting log-likelihood (Eq. 4) must
match the dense oracle (Eq. 1) to the accuracy eps allows."""
import numpy as np
import pytest

from oracle import dense as od
from synthetic import uniform_iid, standard_normal, perturbed_mesh
from plan_interp import Plan, Interp, InterpRand


def _run(tmp_path, pts, theta, leaf, eta, eps, kmax=64, seed=0, k=2, mode="waves", cls=Interp):
    from paper_1709_04419_b200 import Tree
    t = Tree(pts, leaf, eta)
    path = str(tmp_path / "plan.bin")
    t.plan_dump(path, kmax)
    P = Plan(path)
    perm = t.perm()
    I = cls(P, eps, seed=seed, mode=mode)
    I.assemble(pts[perm], theta)
    I.run(P.chol)
    assert I.fail == 0
    z = standard_normal(len(pts), k, seed=5)
    ll, ld, q = I.loglik(z[perm])
    oll, old, oq = od.loglik(pts, z, theta)
    return ll, ld, q, oll, old, oq, I, perm


@pytest.mark.parametrize("n,leaf,eta,eps,seed", [(300, 16, 2.0, 1e-10, 0), (1024, 8, 3.0, 1e-10, 1),
                                                 (777, 16, 1.0, 1e-10, 2), (1000, 32, 2.0, 1e-10, 3)])
def test_planner_matches_dense_oracle(tmp_path, n, leaf, eta, eps, seed):
    pts = uniform_iid(n, seed)
    ll, ld, q, oll, old, oq, _, _ = _run(tmp_path, pts, (1.0, 0.0864, 0.5), leaf, eta, eps, seed=seed)
    np.testing.assert_allclose(ll, oll, rtol=1e-8)
    assert abs(ld - old) <= 1e-6 * abs(old) + 1e-6


@pytest.mark.parametrize("n,leaf,eta,seed", [(600, 16, 2.0, 10), (1024, 8, 3.0, 11)])
def test_planner_dependency_edges(tmp_path, n, leaf, eta, seed):
    """Persistent-executor order: any topological order of xt/xdeps gives the result."""
    pts = uniform_iid(n, seed)
    ll, ld, q, oll, old, oq, _, _ = _run(tmp_path, pts, (1.0, 0.0864, 0.5), leaf, eta, 1e-10, seed=seed, mode="dag")
    np.testing.assert_allclose(ll, oll, rtol=1e-8)
    assert abs(ld - old) <= 1e-6 * abs(old) + 1e-6


@pytest.mark.parametrize("eps,tol", [(1e-10, 1e-9), (1e-7, 1e-5)])
def test_randomized_truncation_algorithm(tmp_path, eps, tol):
    """The device's randomized range-finder truncation (trunc.cuh), replayed with
    numpy on the wide Cholesky truncations, keeps the likelihood at the accuracy
    eps allows (n = 2000, leaf 32: stacked widths reach ~1700 columns).  At
    eps = 1e-10 this needs the second projection of each new block (BCGS2)."""
    pts = uniform_iid(2000, 11)
    ll, ld, q, oll, old, oq, I, _ = _run(tmp_path, pts, (1.0, 0.0864, 0.5), 32, 2.0, eps, kmax=160, seed=0, k=1,
                                         cls=InterpRand)
    np.testing.assert_allclose(ll, oll, rtol=tol)



@pytest.mark.parametrize("eps,tol", [(1e-10, 1e-9), (1e-7, 1e-5)])
def test_split_truncations(tmp_path, monkeypatch, eps, tol):
    """HM_TRUNC_SPLIT=1 (off by default): wide truncations become an early
    partial merge (eps share 1/4) + a final step (3/4); the replayed plan still matches the
    dense oracle at the accuracy eps allows."""
    monkeypatch.setenv("HM_TRUNC_SPLIT", "1")
    pts = uniform_iid(2000, 11)
    ll, ld, q, oll, old, oq, I, _ = _run(tmp_path, pts, (1.0, 0.0864, 0.5), 32, 2.0, eps, kmax=160, seed=0, k=1,
                                         cls=InterpRand)
    np.testing.assert_allclose(ll, oll, rtol=tol)
    P = Plan(str(tmp_path / "plan.bin"))
    sc = P.chol.tt["eps_scale"]
    assert np.any(sc == 0.25) and np.sum(sc == 0.25) == np.sum(sc == 0.75)


def test_randomized_recompression_of_tall_blocks(tmp_path):
    """Recompressions of ACA blocks taller than TR_EXACT_MMAX (512) take the
    cooperative randomized path (hm_tasks.h trunc_exact_path): on a thin strip
    (near 1-D, so 600 x 600 blocks are admissible) the replayed plan still
    matches the dense oracle at the accuracy eps allows."""
    rng = np.random.default_rng(3)
    pts = np.stack([rng.random(2400), 0.01 * rng.random(2400)], axis=1)
    ll, ld, q, oll, old, oq, I, _ = _run(tmp_path, pts, (1.0, 0.2, 0.5), 32, 2.0, 1e-8, kmax=160, seed=0, k=1,
                                         cls=InterpRand)
    P = Plan(str(tmp_path / "plan.bin"))
    tall = [(int(x["m"]), int(x["kmax_tot"])) for x in P.recompress.tt if int(x["m"]) > 512]
    assert tall, "no recompression above TR_EXACT_MMAX in this geometry"
    np.testing.assert_allclose(ll, oll, rtol=1e-6)


def test_planner_general_nu_mesh(tmp_path):
    pts = perturbed_mesh(24, 0.4, seed=4)
    ll, ld, q, oll, old, oq, _, _ = _run(tmp_path, pts, (1.3, 0.2, 1.5), 16, 2.0, 1e-10)
    # smooth field (nu = 3/2, ell = 0.2): C is badly conditioned, error ~ eps * cond
    np.testing.assert_allclose(ll, oll, rtol=1e-6)


def test_planner_error_scales_with_eps(tmp_path):
    pts = uniform_iid(1024, 7)
    errs = []
    for eps in (1e-4, 1e-7, 1e-10):
        ll, _, _, oll, _, _, _, _ = _run(tmp_path, pts, (1.0, 0.1, 0.5), 8, 3.0, eps)
        errs.append(np.max(np.abs(ll - oll) / np.abs(oll)))
    assert errs[0] > errs[1] > errs[2]
    assert errs[2] < 1e-9


def test_sampler_plan_is_L_times_x(tmp_path):
    # lmul phase computes L~ x; with eps tiny, (L~ x) solved back by the solve phase gives x
    pts = uniform_iid(500, 9)
    from paper_1709_04419_b200 import Tree
    t = Tree(pts, 16, 2.0)
    path = str(tmp_path / "plan.bin")
    t.plan_dump(path, 64)
    P = Plan(path)
    perm = t.perm()
    I = Interp(P, 1e-12, seed=1)
    I.assemble(pts[perm], (1.0, 0.1, 0.5))
    I.run(P.chol)
    x = standard_normal(500, 3, seed=2)
    y = I.lmul(x)
    # y y^T ~ C in expectation; exact check: L^{-1} y == x
    I.pool[P.z_off:P.z_off + 500 * P.zw] = 0
    buf = np.zeros((500, P.zw)); buf[:, :3] = y
    I.pool[P.z_off:P.z_off + 500 * P.zw] = buf.ravel(order="F")
    I.run(P.solve)
    back = I.pool[P.z_off:P.z_off + 500 * P.zw].reshape(P.zw, 500).T[:, :3]
    np.testing.assert_allclose(back, x, rtol=1e-9, atol=1e-9)
    # and L~ L~^T == C (dense oracle) through y = L e_j columns
    C = od.covariance(pts[perm], (1.0, 0.1, 0.5))
    E = np.zeros((500, 40)); E[np.arange(40), np.arange(40)] = 1.0
    Lcols = np.concatenate([I.lmul(E[:, i:i + 20]) for i in (0, 20)], axis=1)
    np.testing.assert_allclose(Lcols[:40, :40] @ Lcols[:40, :40].T, C[:40, :40], atol=1e-9)


def test_plan_summary_counts():
    from paper_1709_04419_b200 import Tree
    s = Tree(uniform_iid(2000, 0), 32, 2.0).plan_summary(64)
    assert s["chol_waves"] > 0 and s["chol_vm_tasks"] > 0 and s["solve_tasks"] > 0


@pytest.mark.parametrize("n,leaf,eps,seed", [(65, 32, 1e-10, 20), (1040, 32, 1e-10, 21), (1500, 100, 1e-10, 22),
                                             (2000, 128, 1e-9, 23), (777, 48, 1e-10, 24)])
def test_mixed_depth_and_large_leaves(tmp_path, n, leaf, eps, seed):
    """General n (Def. 1 l.152-160 and n_min l.211 put no restriction on n;
    Table 1 l.213 allows n_min up to 128): when n / 2^l straddles n_min the tree has
    leaves at two depths (65 points, leaf 32: 32 | 33 -> 16/17), and leaves above 64
    exceed one tile.  The planner runs on the refined storage tree (tree.h
    refine_for_plan) -- the DAG replayed in random wave order must still match the
    dense oracle, while the exported tree and partition stay the oracle's (bit-exact,
    test_abi_host.py)."""
    from paper_1709_04419_b200 import Tree
    from oracle import geometry as og
    pts = uniform_iid(n, seed)
    t = Tree(pts, leaf, 2.0)
    levels = {int(c[2]) for c in t.clusters() if c[3]}
    big = max(int(c[1] - c[0]) for c in t.clusters() if c[3])
    assert len(levels) > 1 or big > 64, "case must exercise the storage refinement"
    ll, ld, q, oll, old, oq, _, _ = _run(tmp_path, pts, (1.0, 0.0864, 0.5), leaf, 2.0, eps, seed=seed)
    np.testing.assert_allclose(ll, oll, rtol=1e-8)
    assert abs(ld - old) <= 1e-6 * abs(old) + 1e-6


def test_paper_table2_size_plans():
    """PAPER.md Table 2 (l.228-249): n = 16,641 on the perturbed mesh (Eq. 3) at
    n_min = 32 (l.211), and configs[2]'s size + 1 at leaf 64: both plan (they
    were rejected before the storage refinement)."""
    from paper_1709_04419_b200 import Tree
    s = Tree(perturbed_mesh(129, 0.4, seed=5), 32, 2.0).plan_summary(64)
    assert s["chol_vm_tasks"] > 0 and s["solve_tasks"] > 0
    s = Tree(uniform_iid(65537, 6), 64, 2.0).plan_summary(64)
    assert s["chol_vm_tasks"] > 0


def test_ready_queue_schedule_replays_on_host():
    """The persistent executor's ready-queue schedule (sched.cpp: successor lists,
    arrival counts, priority queues, cooperative groups pushed as consecutive slots)
    is built for every phase of the plan and its host replay must reach every task
    exactly once with every queue sized exactly (hm_plan_dump raises otherwise) --
    checked here without a GPU, on a plan with cooperative truncations."""
    from paper_1709_04419_b200 import Tree
    s = Tree(uniform_iid(4096, 3), 32, 2.0).plan_summary(64)
    assert s["chol_trunc_tasks"] > 0
