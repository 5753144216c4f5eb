"""Multi-GPU sharding of independent likelihood evaluations (host logic only).

The north star partitions the work only where it shards naturally: independent
theta points of an MLE search / grid and Monte-Carlo replicates.  A single
factorisation stays on one GPU.  Each rank (one process per GPU,
torch.distributed) evaluates its own slice of the theta list through the C-ABI
(``hm_loglik_batch``) and the (loglik, logdet, quad) triples are gathered once
at the end -- there is no collective on the data path.

The functions here are pure host logic (slicing + one all_gather) so they are
tested with the gloo backend on CPU (tests/test_dist_gloo.py); on the GPU box
the same code runs over NCCL.
"""
from __future__ import annotations

import numpy as np


def shard_indices(n_items: int, rank: int, world: int) -> np.ndarray:
    """Round-robin slice of range(n_items) owned by ``rank`` (balanced to +-1)."""
    if not (0 <= rank < world):
        raise ValueError("0 <= rank < world required")
    return np.arange(rank, n_items, world, dtype=np.int64)


def gather_results(local: np.ndarray, n_items: int, rank: int, world: int, device=None) -> np.ndarray:
    """All-gather per-item result rows computed on each rank's shard.

    local: (len(shard_indices(n_items, rank, world)), ...) float64 rows in shard
    order.  Returns the (n_items, ...) array in the original item order on every
    rank.  One all_gather of equal-sized (padded) tensors.
    """
    import torch
    import torch.distributed as dist

    local = np.ascontiguousarray(local, dtype=np.float64)
    tail = local.shape[1:]
    per = (n_items + world - 1) // world
    buf = np.full((per,) + tail, np.nan)
    buf[: local.shape[0]] = local
    t = torch.from_numpy(buf)
    if device is None and dist.get_backend() == "nccl":   # NCCL moves device tensors only
        device = torch.device("cuda", torch.cuda.current_device())
    if device is not None:
        t = t.to(device)
    parts = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(parts, t)
    out = np.empty((n_items,) + tail)
    for r in range(world):
        idx = shard_indices(n_items, r, world)
        out[idx] = parts[r].cpu().numpy()[: idx.size]
    return out


def loglik_sharded(H, thetas, Z, rank: int, world: int, device=None):
    """Evaluate Eq. (4) for this rank's slice of ``thetas`` on handle H (one GPU)
    and gather every rank's results: returns (n_theta, k, 3) and the first
    non-zero status code seen locally (0 if none)."""
    thetas = np.asarray(thetas, dtype=np.float64).reshape(-1, 3)
    idx = shard_indices(thetas.shape[0], rank, world)
    if idx.size:
        out, rc = H.loglik_batch(thetas[idx], Z)
    else:
        k = 1 if np.ndim(Z) == 1 else (Z.shape[1] if hasattr(Z, "shape") else 1)
        out, rc = np.zeros((0, k, 3)), 0
    return gather_results(out, thetas.shape[0], rank, world, device=device), rc
