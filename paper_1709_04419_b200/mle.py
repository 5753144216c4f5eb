"""Maximum-likelihood driver (BASELINE configs[3]: Monte-Carlo MLE).

PAPER.md sec. 3.1 (l.256-270): theta-hat maximises Eq. (4); the paper uses a
Brent-Dekker line search (l.268) and, in sec. 4-5, estimates (ell, nu, sigma^2)
jointly.  configs[3] fixes the optimiser's budget: every replicate runs exactly
`evals` likelihood evaluations of a Nelder-Mead search over
(log sigma^2, log ell, log nu) -- the log map keeps theta > 0 (Eq. 2 domain).

Only the likelihood evaluations are the hot path (hm_assemble + hm_cholesky +
hm_loglik through the C-ABI on the GPU); the simplex bookkeeping is host logic
and is tested on the CPU (tests/test_mle.py).  Replicates are sharded over
ranks with paper_1709_04419_b200.dist (no data-path collective).
"""
from __future__ import annotations

import math

import numpy as np

from .dist import gather_results, shard_indices


def nelder_mead(f, x0, step, evals: int):
    """Minimise f over R^d with exactly `evals` evaluations of f (standard
    reflection/expansion/contraction/shrink coefficients 1, 2, 1/2, 1/2).
    Returns (x_best, f_best, history) with history = [(x, f(x)), ...]."""
    x0 = np.asarray(x0, dtype=np.float64)
    d = x0.size
    hist = []

    def ev(x):
        if len(hist) >= evals:
            raise StopIteration
        v = float(f(x))
        if not math.isfinite(v):
            v = math.inf
        hist.append((x.copy(), v))
        return v

    try:
        simplex = [x0.copy()] + [x0 + step * np.eye(d)[i] for i in range(d)]
        vals = [ev(x) for x in simplex]
        while True:
            order = np.argsort(vals)
            simplex = [simplex[i] for i in order]
            vals = [vals[i] for i in order]
            c = np.mean(simplex[:-1], axis=0)
            xr = c + (c - simplex[-1])
            fr = ev(xr)
            if vals[0] <= fr < vals[-2]:
                simplex[-1], vals[-1] = xr, fr
                continue
            if fr < vals[0]:
                xe = c + 2.0 * (c - simplex[-1])
                fe = ev(xe)
                if fe < fr:
                    simplex[-1], vals[-1] = xe, fe
                else:
                    simplex[-1], vals[-1] = xr, fr
                continue
            if fr < vals[-1]:                     # outside contraction
                xc = c + 0.5 * (xr - c)
                fc = ev(xc)
                if fc <= fr:
                    simplex[-1], vals[-1] = xc, fc
                    continue
            else:                                 # inside contraction
                xc = c + 0.5 * (simplex[-1] - c)
                fc = ev(xc)
                if fc < vals[-1]:
                    simplex[-1], vals[-1] = xc, fc
                    continue
            for i in range(1, d + 1):             # shrink towards the best vertex
                simplex[i] = simplex[0] + 0.5 * (simplex[i] - simplex[0])
                vals[i] = ev(simplex[i])
    except StopIteration:
        pass
    best = min(hist, key=lambda h: h[1])
    return best[0], best[1], hist


def mle_replicate(H, Z, theta0, evals: int = 60, step: float = 0.3):
    """Nelder-Mead on -loglik(theta) (Eq. 4) over log-parameters for one replicate
    (handle H on its locations, data Z).  A theta whose H-Cholesky fails
    (HM_ERR_NOT_SPD, reading R9) scores +inf.  Returns (theta_hat, loglik_hat, n_evals)."""
    from ._binding import HMError

    def negll(x):
        th = tuple(float(v) for v in np.exp(x))
        try:
            H.assemble(th)
            H.cholesky()
            return -float(H.loglik(Z)[0, 0])
        except HMError:
            return math.inf

    x, fx, hist = nelder_mead(negll, np.log(np.asarray(theta0, dtype=np.float64)), step, evals)
    return np.exp(x), -fx, len(hist)


class _LockstepBatcher:
    """Runs S Nelder-Mead searches in lockstep: each search (its own host thread)
    posts its next theta and waits; when every live search has posted, ONE
    hm_loglik_multi call evaluates them all co-scheduled on the GPU (C-ABI,
    include/hmlik.h) and hands the results back.  The searches stay in step
    because each spends exactly the same budget of evaluations."""

    def __init__(self, handles, Zs):
        import threading
        self.H, self.Z = handles, Zs
        self.live = len(handles)
        self.req = {}
        self.res = {}
        self.cv = threading.Condition()
        self.gen = 0

    def _flush(self):
        from ._binding import loglik_multi
        idx = sorted(self.req)
        out, _ = loglik_multi([self.H[i] for i in idx], [self.req[i] for i in idx], [self.Z[i] for i in idx])
        for j, i in enumerate(idx):
            v = out[j, 0, 0]
            self.res[i] = -float(v) if math.isfinite(v) else math.inf
        self.req.clear()
        self.gen += 1
        self.cv.notify_all()

    def negll(self, i, x):
        th = tuple(float(v) for v in np.exp(x))
        with self.cv:
            self.req[i] = th
            g = self.gen
            if len(self.req) == self.live:
                self._flush()
            while self.gen == g:
                self.cv.wait()
            return self.res.pop(i)

    def done(self):
        with self.cv:
            self.live -= 1
            if self.live > 0 and len(self.req) == self.live:
                self._flush()


def mc_mle(n: int, replicates: int, theta_true, theta0, eps: float = 1e-6, evals: int = 60, leaf: int = 32,
           eta: float = 2.0, rank: int = 0, world: int = 1, device: int = 0, seed: int = 0, gather: bool = True,
           streams: int = 1, sms: int = 148, kmax: int = 0):
    """configs[3]: `replicates` independent data sets (n uniform iid locations in
    [0,1]^2, Z = L~(theta_true) xi drawn by the library's H-sampler at min(eps, 1e-8)),
    each fitted by `evals` Nelder-Mead evaluations.  Replicates are sharded
    round-robin over ranks; returns (replicates x 5): sigma2, ell, nu, loglik, evals.

    streams = S > 1: the rank's replicates are fitted S at a time, their searches in
    lockstep, every round of S likelihood evaluations ONE hm_loglik_multi call
    (S handles co-scheduled behind the C-ABI, each executor on sms / S CTAs,
    cooperative truncation groups sized to fit that share); the results equal the
    one-at-a-time run on the same plan (the CTA cap never changes the arithmetic)."""
    import threading

    from ._binding import HMatrix
    from synthetic import standard_normal, uniform_iid

    mine = list(shard_indices(replicates, rank, world))
    S = max(1, int(streams))
    cap = sms // S if S > 1 else 0
    # deadlock bound of the ready-queue executor: 4 * (coop - 1) < CTAs per executor
    coop = 16 if S == 1 else max(1, min(8, (cap - 1) // 4 + 1))
    kw = dict(leaf=leaf, eta=eta, device=device, kmax=kmax, coop_max=coop, exec_ctas=cap)
    res = {}

    def data(r):
        pts = uniform_iid(n, seed + 1000 * int(r))
        Hs = HMatrix(pts, theta_true, eps=min(eps, 1e-8), **kw)
        Hs.cholesky()
        Z = Hs.sample(standard_normal(n, 1, seed + 1000 * int(r) + 1))[:, 0]
        Hs.close()
        return pts, Z

    for g0 in range(0, len(mine), S):
        group = mine[g0:g0 + S]
        sets = [data(r) for r in group]
        Hs = [HMatrix(p, theta0, eps=eps, **kw) for p, _ in sets]
        if len(group) == 1:
            th, ll, ne = mle_replicate(Hs[0], sets[0][1], theta0, evals=evals)
            res[group[0]] = [th[0], th[1], th[2], ll, ne]
        else:
            B = _LockstepBatcher(Hs, [Z for _, Z in sets])
            errs = []

            def search(i, r):
                try:
                    x, fx, hist = nelder_mead(lambda x: B.negll(i, x), np.log(np.asarray(theta0, dtype=np.float64)),
                                              0.3, evals)
                    th = np.exp(x)
                    res[r] = [th[0], th[1], th[2], -fx, len(hist)]
                except Exception as e:  # surfaced after the join
                    errs.append(e)
                finally:
                    B.done()

            ts = [threading.Thread(target=search, args=(i, r)) for i, r in enumerate(group)]
            for t in ts:
                t.start()
            for t in ts:
                t.join()
            if errs:
                raise errs[0]
        for H in Hs:
            H.close()
    out = [res[r] for r in mine]
    local = np.asarray(out, dtype=np.float64).reshape(-1, 5)
    if world > 1 and gather:
        return gather_results(local, replicates, rank, world)
    return local
