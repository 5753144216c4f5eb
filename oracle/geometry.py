"""Oracle: cluster tree and block cluster tree (sec. 2.1).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md l.143-145: "hierarchical partitioning of a given matrix into
sub-blocks ... a so-called admissibility condition is used".  Definition 1
(l.152-160) defines H(T_{IxI}, k) over the block cluster tree T_{IxI}; l.211
gives the leaf size n_min ("Usually n_min = 32 or 64").  The paper states
neither the splitting rule nor the admissibility condition; DESIGN.md sec. 3
fixes our readings, which this file follows literally:

R1  a cluster t with |t| > n_min is split at the median of its points along
    the longest axis of its tight bounding box (first axis on ties); points
    are ordered by (coordinate, original index); the first floor(|t|/2) go to
    the first child.
R2  block (t, s) is admissible iff dist(t, s) > 0 and
    min(diam t, diam s) <= eta * dist(t, s), diam/dist computed on the tight
    axis-aligned bounding boxes as sqrt(dx*dx + dy*dy) in IEEE double, left to
    right (dist > 0 keeps every block that meets the diagonal dense, also for
    degenerate single-point clusters whose diam is 0).
R3  a non-admissible block becomes a dense leaf if t or s is a leaf cluster,
    otherwise it is subdivided into the four children pairs.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np


@dataclass
class Cluster:
    lo: int                 # index range [lo, hi) in the permuted ordering
    hi: int
    level: int
    bmin: tuple             # (xmin, ymin)
    bmax: tuple             # (xmax, ymax)
    children: list = field(default_factory=list)

    @property
    def size(self) -> int:
        return self.hi - self.lo

    @property
    def is_leaf(self) -> bool:
        return not self.children


def build_cluster_tree(points: np.ndarray, n_min: int):
    """R1.  Returns (root, perm) with perm[k] = original index of the k-th point
    in tree order (so points[perm] is the tree-ordered set)."""
    pts = np.asarray(points, dtype=np.float64)
    if pts.ndim != 2 or pts.shape[1] != 2:
        raise ValueError("points must be n x 2")
    n = pts.shape[0]
    if n < 1:
        raise ValueError("empty point set")
    if n_min < 1:
        raise ValueError("n_min >= 1 required")
    if not np.all(np.isfinite(pts)):
        raise ValueError("non-finite coordinate")
    perm = np.arange(n, dtype=np.int64)

    def rec(lo: int, hi: int, level: int) -> Cluster:
        idx = perm[lo:hi]
        sub = pts[idx]
        bmin = (float(sub[:, 0].min()), float(sub[:, 1].min()))
        bmax = (float(sub[:, 0].max()), float(sub[:, 1].max()))
        node = Cluster(lo, hi, level, bmin, bmax)
        m = hi - lo
        if m > n_min:
            ext0 = bmax[0] - bmin[0]
            ext1 = bmax[1] - bmin[1]
            axis = 0 if ext0 >= ext1 else 1
            order = np.lexsort((idx, sub[:, axis]))   # primary: coord, then original index
            perm[lo:hi] = idx[order]
            mid = lo + m // 2
            node.children = [rec(lo, mid, level + 1), rec(mid, hi, level + 1)]
        return node

    root = rec(0, n, 0)
    return root, perm


def diameter(c: Cluster) -> float:
    dx = c.bmax[0] - c.bmin[0]
    dy = c.bmax[1] - c.bmin[1]
    return math.sqrt(dx * dx + dy * dy)


def distance(t: Cluster, s: Cluster) -> float:
    dx = max(0.0, s.bmin[0] - t.bmax[0], t.bmin[0] - s.bmax[0])
    dy = max(0.0, s.bmin[1] - t.bmax[1], t.bmin[1] - s.bmax[1])
    return math.sqrt(dx * dx + dy * dy)


def admissible(t: Cluster, s: Cluster, eta: float) -> bool:
    """R2."""
    d = distance(t, s)
    return d > 0.0 and min(diameter(t), diameter(s)) <= eta * d


def build_block_partition(root: Cluster, eta: float):
    """R2 + R3 over the full index set I x I.  Returns the leaf blocks as a list
    of tuples (t_lo, t_hi, s_lo, s_hi, level, admissible_flag)."""
    if not eta > 0:
        raise ValueError("eta > 0 required")
    out = []

    def rec(t: Cluster, s: Cluster):
        if admissible(t, s, eta):
            out.append((t.lo, t.hi, s.lo, s.hi, t.level, 1))
        elif t.is_leaf or s.is_leaf:
            out.append((t.lo, t.hi, s.lo, s.hi, t.level, 0))
        else:
            for tc in t.children:
                for sc in s.children:
                    rec(tc, sc)

    rec(root, root)
    return out


def tree_nodes(root: Cluster):
    """Pre-order list of (lo, hi, level, is_leaf) -- used for bit-exact comparison."""
    out = []
    stack = [root]
    while stack:
        c = stack.pop()
        out.append((c.lo, c.hi, c.level, int(c.is_leaf)))
        stack.extend(reversed(c.children))
    return out
