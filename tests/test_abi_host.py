"""Host-only checks of the C-ABI library (no GPU needed): the .so loads, exports
every symbol include/hmlik.h declares, and its host geometry (cluster tree +
block partition, sec. 2.1) is bit-exact against the oracle."""
import ctypes
import os
import re

import numpy as np
import pytest

from oracle.geometry import build_cluster_tree, build_block_partition, tree_nodes
from synthetic import uniform_iid, perturbed_mesh, latlon_dropout

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "hmlik.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(hm_\w+)\s*\(", src, re.M)))


def test_library_exports_every_declared_symbol():
    from paper_1709_04419_b200 import _binding
    lib = ctypes.CDLL(_binding.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_binding.EXPORTED)
    assert b"sm_100a" in _binding.lib.hm_version()


def _compare(pts, leaf, eta):
    from paper_1709_04419_b200 import Tree
    t = Tree(pts, leaf, eta)
    root, perm = build_cluster_tree(pts, leaf)
    assert np.array_equal(t.perm(), perm)
    assert [tuple(r) for r in t.clusters().tolist()] == tree_nodes(root)
    ob = build_block_partition(root, eta)
    gb = [tuple(r) for r in t.blocks().tolist()]
    assert gb == ob                         # same blocks, same order, same flags
    assert t.n_admissible == sum(b[5] for b in ob)
    return t


@pytest.mark.parametrize("n,leaf,eta,seed", [(1, 32, 2.0, 0), (2, 1, 2.0, 1), (64, 32, 2.0, 2),
                                             (2000, 32, 2.0, 3), (4097, 64, 2.0, 4), (3000, 7, 0.7, 5)])
def test_tree_bit_exact_uniform(n, leaf, eta, seed):
    _compare(uniform_iid(n, seed), leaf, eta)


def test_tree_bit_exact_config2_mesh():
    # configs[2] geometry: 256 x 256 jittered grid, leaf 64 (Eq. 3 with delta = 0.4)
    _compare(perturbed_mesh(256, 0.4, seed=2), 64, 2.0)


def test_tree_bit_exact_ties():
    # duplicate coordinates exercise the (coordinate, original index) tie-break
    pts = np.round(uniform_iid(3000, 9) * 8) / 8
    _compare(pts, 16, 2.0)


def test_tree_bit_exact_latlon_small():
    _compare(latlon_dropout(5000, seed=4, h=0.1), 32, 2.0)


def test_tree_errors():
    from paper_1709_04419_b200 import Tree, HMError
    with pytest.raises(HMError):
        Tree(np.zeros((0, 2)), 32, 2.0)
    with pytest.raises(HMError):
        Tree(np.array([[0.0, np.nan]]), 32, 2.0)
    with pytest.raises(HMError):
        Tree(uniform_iid(10, 0), 32, 0.0)
