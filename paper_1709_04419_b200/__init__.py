"""B200-native H-matrix Gaussian log-likelihood (arxiv 1709.04419 hot path).

Public Python API = thin wrappers over the C-ABI in include/hmlik.h:
``Tree``, ``HMatrix`` (hm_build / hm_cholesky / hm_loglik / ...),
``dense_loglik`` (GPU dense check path), ``matern_block``.
"""
from ._binding import (HMError, HMatrix, Tree, dense_loglik, loglik_multi, matern_block, lib)  # noqa: F401

__all__ = ["HMError", "HMatrix", "Tree", "dense_loglik", "loglik_multi", "matern_block", "lib"]
