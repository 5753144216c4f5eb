"""Pins for oracle.geometry (sec. 2.1, Definition 1, l.152-160; l.211).

Checks that do not reuse the oracle's own code path: hand-built partitions,
an independent size-only recursion for node/leaf counts, exhaustive tiling of
I x I, bounding boxes and admissibility recomputed from the raw points with
numpy reductions, and the median-split ordering property.
"""
import math

import numpy as np
import pytest

from oracle.geometry import (build_cluster_tree, build_block_partition, tree_nodes)
from synthetic import uniform_iid, perturbed_mesh


def all_clusters(root):
    out, st = [], [root]
    while st:
        c = st.pop()
        out.append(c)
        st.extend(c.children)
    return out


def test_single_point():
    root, perm = build_cluster_tree(np.array([[0.5, 0.5]]), 32)
    assert root.is_leaf and root.size == 1 and list(perm) == [0]
    blocks = build_block_partition(root, 2.0)
    assert blocks == [(0, 1, 0, 1, 0, 0)]


def test_collinear_64_forced_median_split():
    x = np.linspace(1.0, 0.0, 64)             # reversed so the permutation is non-trivial
    pts = np.stack([x, np.zeros(64)], axis=1)
    root, perm = build_cluster_tree(pts, 32)
    assert [c.size for c in root.children] == [32, 32]
    assert all(c.is_leaf for c in root.children)
    left = pts[perm[:32]]
    right = pts[perm[32:]]
    assert left[:, 0].max() < right[:, 0].min()   # split along the line's axis
    assert list(perm[:32]) == list(range(63, 31, -1))


def size_only_counts(n, n_min):
    """Independent recursion on sizes only: (#nodes, #leaves, depth)."""
    if n <= n_min:
        return 1, 1, 0
    a = size_only_counts(n // 2, n_min)
    b = size_only_counts(n - n // 2, n_min)
    return 1 + a[0] + b[0], a[1] + b[1], 1 + max(a[2], b[2])


@pytest.mark.parametrize("n,n_min", [(16641, 32), (2000, 32), (4096, 64), (1000, 7)])
def test_counts_match_size_recursion(n, n_min):
    pts = perturbed_mesh(129, 0.4, seed=1)[:n] if n <= 16641 else None
    root, perm = build_cluster_tree(pts, n_min)
    nodes = tree_nodes(root)
    nn, nl, depth = size_only_counts(n, n_min)
    assert len(nodes) == nn
    assert sum(1 for t in nodes if t[3]) == nl
    assert max(t[2] for t in nodes) == depth
    assert depth <= math.ceil(math.log2(max(n / n_min, 1))) + 1
    assert sorted(perm.tolist()) == list(range(n))


def test_tree_invariants_from_raw_points():
    pts = uniform_iid(1500, seed=42)
    root, perm = build_cluster_tree(pts, 20)
    for c in all_clusters(root):
        sub = pts[perm[c.lo:c.hi]]
        assert c.bmin == (sub[:, 0].min(), sub[:, 1].min())
        assert c.bmax == (sub[:, 0].max(), sub[:, 1].max())
        if c.is_leaf:
            assert c.size <= 20
        else:
            a, b = c.children
            assert (a.lo, a.hi, b.lo, b.hi) == (c.lo, c.lo + c.size // 2, c.lo + c.size // 2, c.hi)
            ext = np.ptp(sub, axis=0)
            axis = 0 if ext[0] >= ext[1] else 1
            ia, ib = perm[a.lo:a.hi], perm[b.lo:b.hi]
            key = lambda i: (pts[i, axis], i)
            assert max(map(key, ia)) < min(map(key, ib))   # median split along the longest axis


def box_of(pts):
    return pts.min(axis=0), pts.max(axis=0)


def test_partition_tiles_and_admissibility_exhaustive():
    n, n_min, eta = 900, 16, 2.0
    pts = uniform_iid(n, seed=8)
    root, perm = build_cluster_tree(pts, n_min)
    blocks = build_block_partition(root, eta)
    cover = np.zeros((n, n), dtype=np.int32)
    leaves = {(c.lo, c.hi) for c in all_clusters(root) if c.is_leaf}
    for (tlo, thi, slo, shi, lev, adm) in blocks:
        cover[tlo:thi, slo:shi] += 1
        tp, sp = pts[perm[tlo:thi]], pts[perm[slo:shi]]
        (tmin, tmax), (smin, smax) = box_of(tp), box_of(sp)
        dt, ds = np.hypot(*(tmax - tmin)), np.hypot(*(smax - smin))
        gap = np.maximum(0, np.maximum(smin - tmax, tmin - smax))
        dist = np.hypot(*gap)
        if adm:
            assert min(dt, ds) <= eta * dist * (1 + 1e-12)
            assert dist > 0
        else:
            assert min(dt, ds) > eta * dist * (1 - 1e-12)
            assert (tlo, thi) in leaves or (slo, shi) in leaves
    assert np.all(cover == 1)                                # leaf blocks tile I x I exactly once
    # symmetry of the partition
    s = {(b[0], b[1], b[2], b[3], b[5]) for b in blocks}
    assert all((b[2], b[3], b[0], b[1], b[5]) in s for b in blocks)


def test_hand_built_line_partition():
    # points 0,1,2,3 and 10,11,12,13 on the x axis, n_min = 2.
    xs = np.array([13, 0, 12, 1, 11, 2, 10, 3], dtype=float)
    pts = np.stack([xs, np.zeros(8)], axis=1)
    root, perm = build_cluster_tree(pts, 2)
    assert pts[perm, 0].tolist() == [0, 1, 2, 3, 10, 11, 12, 13]
    # eta = 1: halves have diam 3, dist 7 -> admissible; quarters {0,1},{2,3} diam 1 dist 1 -> admissible
    got = sorted(build_block_partition(root, 1.0))
    want = sorted([
        (0, 4, 4, 8, 1, 1), (4, 8, 0, 4, 1, 1),
        (0, 2, 2, 4, 2, 1), (2, 4, 0, 2, 2, 1), (4, 6, 6, 8, 2, 1), (6, 8, 4, 6, 2, 1),
        (0, 2, 0, 2, 2, 0), (2, 4, 2, 4, 2, 0), (4, 6, 4, 6, 2, 0), (6, 8, 6, 8, 2, 0),
    ])
    assert got == want
    # eta = 0.9: quarters no longer admissible (1 > 0.9), halves still are (3 <= 6.3)
    got = sorted(build_block_partition(root, 0.9))
    want2 = [b if b[4] == 1 else b for b in want]
    want2 = sorted([(a, b, c, d, l, 1 if l == 1 else 0) for (a, b, c, d, l, _) in want])
    assert got == want2


def test_touching_clusters_inadmissible():
    pts = perturbed_mesh(16, 0.0, seed=0)        # regular lattice: siblings always touch
    root, _ = build_cluster_tree(pts, 8)
    for (tlo, thi, slo, shi, lev, adm) in build_block_partition(root, 2.0):
        if adm:
            assert not (tlo < shi and slo < thi)   # never overlapping ranges
    a, b = root.children
    from oracle.geometry import admissible, distance
    assert not admissible(a, b, 2.0)
    assert not admissible(a, a, 2.0) and distance(a, a) == 0.0


def test_perturbed_mesh_eq3():
    p = perturbed_mesh(2, 0.0, seed=0)
    assert p.tolist() == [[0.25, 0.25], [0.25, 0.75], [0.75, 0.25], [0.75, 0.75]]
    q = perturbed_mesh(129, 0.4, seed=3)
    assert q.shape == (16641, 2) and q.min() > 0 and q.max() < 1
    assert np.array_equal(q, perturbed_mesh(129, 0.4, seed=3))
