"""Multi-process (world_size 2, gloo, CPU) test of the theta/replicate sharding
used for the batched evaluations (paper_1709_04419_b200/dist.py): every theta
is evaluated exactly once, by its owner rank, and every rank ends with all
results in the original order."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


class FakeHandle:
    """Stands in for HMatrix on CPU: a deterministic function of theta."""

    def __init__(self, rank):
        self.rank = rank
        self.calls = []

    def loglik_batch(self, thetas, Z):
        thetas = np.asarray(thetas)
        self.calls.extend(map(tuple, thetas))
        k = Z.shape[1]
        out = np.empty((thetas.shape[0], k, 3))
        for i, th in enumerate(thetas):
            for c in range(k):
                out[i, c] = (th[0] + 10 * th[1] + 100 * th[2] + c, float(self.rank), th.sum())
        return out, 0


def _worker(rank, world, port, n_theta, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1709_04419_b200.dist import loglik_sharded, shard_indices
    rng = np.random.default_rng(0)
    thetas = rng.random((n_theta, 3)) + 0.1
    Z = np.zeros((7, 2))
    H = FakeHandle(rank)
    out, rc = loglik_sharded(H, thetas, Z, rank, world)
    q.put((rank, out, H.calls, shard_indices(n_theta, rank, world).tolist(), rc))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("n_theta", [7, 8, 1])
def test_sharded_evaluation_world2(n_theta):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_theta, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda r: r[0])
    rng = np.random.default_rng(0)
    thetas = rng.random((n_theta, 3)) + 0.1
    owners = np.empty(n_theta)
    seen = []
    for rank, out, calls, idx, rc in res:
        assert rc == 0
        assert out.shape == (n_theta, 2, 3)
        owners[idx] = rank
        seen.extend(idx)
        np.testing.assert_array_equal(np.array(calls).reshape(-1, 3), thetas[idx])
    assert sorted(seen) == list(range(n_theta))            # each theta exactly once
    for rank, out, *_ in res:                                # identical, original order, on every rank
        np.testing.assert_array_equal(out, res[0][1])
        np.testing.assert_allclose(out[:, 0, 0], thetas[:, 0] + 10 * thetas[:, 1] + 100 * thetas[:, 2])
        np.testing.assert_array_equal(out[:, 1, 1], owners)



def _bench_worker(rank, world, port, q):
    """bench.py's rank logic on CPU: each rank's theta slice (rank_thetas) and the
    gather of the per-evaluation (loglik, logdet, quad) triples after the timed region."""
    import sys
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import bench
    from paper_1709_04419_b200.dist import gather_results
    w = bench.WORKLOADS["n64k"]
    S, steps = 4, 3
    mine = bench.rank_thetas(w, steps, S, rank, world)
    res = np.array([[th[1], th[2], float(rank)] for th in mine])   # stands in for loglik_batch output
    allres = gather_results(res, len(res) * world, rank, world)
    q.put((rank, mine, allres))
    dist.barrier()
    dist.destroy_process_group()


def test_bench_rank_logic_world2():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bench_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in range(world)], key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    full = bench.theta_schedule(bench.WORKLOADS["n64k"], 3 * 2 * 4)
    got = sorted(tuple(th) for r in res for th in r[1])
    assert got == sorted(map(tuple, full)) and len(res[0][1]) == len(res[1][1]) == 12   # disjoint, complete
    np.testing.assert_array_equal(res[0][2], res[1][2])                               # same gathered table
    assert sorted(res[0][2][:, 2].tolist()) == [0.0] * 12 + [1.0] * 12                 # every rank's rows
