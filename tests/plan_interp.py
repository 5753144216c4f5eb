"""Test-only CPU interpreter of the H-Cholesky task DAG (host planner output).

It executes the tasks that ``hm_plan_dump`` writes -- the exact programs the
GPU tile VM and truncation kernel run -- with numpy, visiting the tasks of
each wave in a RANDOM order.  Comparing its log-likelihood with the dense
oracle therefore checks the planner's H-arithmetic (update bookkeeping,
pushes, products, truncation pieces) and its dependency analysis (a missing
edge inside a wave shows up as an order-dependent wrong answer) without a GPU.

Block entries and the initial low-rank factors come from ``oracle`` (dense
Matern blocks + exact truncated SVD), not from the CUDA kernels: this file
validates host logic only and is never reachable from the product path.
"""
from __future__ import annotations

import math

import numpy as np
import scipy.linalg

from oracle.matern import matern

DIM = np.dtype([("stat", "<i4"), ("slot", "<i4"), ("off", "<i4"), ("pad", "<i4")])
VINS = np.dtype([("op", "u1"), ("t0", "u1"), ("t1", "u1"), ("t2", "u1"), ("ta", "u1"), ("tb", "u1"),
                 ("p0", "u1"), ("p1", "u1"), ("rows", DIM), ("cols", DIM), ("goff", "<i8"), ("ld", "<i4"),
                 ("p2", "<i4"), ("alpha", "<f8"), ("beta", "<f8")])
VTASK = np.dtype([("ins_begin", "<i4"), ("ins_count", "<i4")])
TTASK = np.dtype([("u_out", "<i8"), ("v_out", "<i8"), ("ws", "<i8"), ("ws_size", "<i8"), ("m", "<i4"),
                  ("q", "<i4"), ("cap", "<i4"), ("rslot", "<i4"), ("piece_begin", "<i4"), ("piece_count", "<i4"),
                  ("kmax_tot", "<i4"), ("wmax", "<i4"), ("nsub", "<i4"), ("bar", "<i4"), ("eps_scale", "<f8")])
TPIECE = np.dtype([("u_off", "<i8"), ("v_off", "<i8"), ("u_ld", "<i4"), ("v_ld", "<i4"), ("u_row0", "<i4"),
                   ("u_rows", "<i4"), ("v_row0", "<i4"), ("v_rows", "<i4"), ("w", DIM), ("alpha", "<f8")])
DGEN = np.dtype([("off", "<i8"), ("r0", "<i4"), ("c0", "<i4"), ("m", "<i4"), ("q", "<i4")])
ACA = np.dtype([("u_off", "<i8"), ("v_off", "<i8"), ("r0", "<i4"), ("c0", "<i4"), ("m", "<i4"), ("q", "<i4"),
                ("cap", "<i4"), ("rslot", "<i4")])

VM_LD, VM_ST, VM_GEMM, VM_POTRF, VM_TRSM_RLT, VM_TRSM_LN, VM_TRMM_LN, VM_ZERO, VM_MGEMM, VM_TRTRI, VM_ADD, \
    VM_MGEMM_ST = range(1, 13)
TD = 64


def _read(path):
    raw = open(path, "rb").read()
    pos = 0
    out = []
    while pos < len(raw):
        cnt, size = np.frombuffer(raw, "<i8", 2, pos)
        pos += 16
        out.append((int(cnt), int(size), raw[pos:pos + cnt * size]))
        pos += cnt * size
    return out


VTERM = np.dtype([("a_off", "<i8"), ("b_off", "<i8"), ("a_rows", DIM), ("a_cols", DIM), ("b_rows", DIM),
                  ("b_cols", DIM), ("a_ld", "<i4"), ("b_ld", "<i4"), ("ta", "u1"), ("tb", "u1"), ("p", "u1", (6,)),
                  ("alpha", "<f8")])
XTASK = np.dtype([("kind", "<i4"), ("idx", "<i4"), ("dep_begin", "<i4"), ("dep_count", "<i4"), ("sub", "<i4"),
                  ("nsub", "<i4")])


class Phase:
    def __init__(self, secs):
        (ni, si, bi), (nv, sv, bv), (nt, st, bt), (np_, sp, bp), (nw1, _, bw1), (nw2, _, bw2), (nx, sx, bx), \
            (nd, _, bd), (nm, sm_, bm) = secs
        assert sx == XTASK.itemsize and (nm == 0 or sm_ == VTERM.itemsize)
        self.terms = np.frombuffer(bm, VTERM, nm)
        self.xt = np.frombuffer(bx, XTASK, nx)
        self.xdeps = np.frombuffer(bd, "<i4", nd)
        assert si == VINS.itemsize and sv == VTASK.itemsize and st == TTASK.itemsize and sp == TPIECE.itemsize
        self.ins = np.frombuffer(bi, VINS, ni)
        self.vt = np.frombuffer(bv, VTASK, nv)
        self.tt = np.frombuffer(bt, TTASK, nt)
        self.tp = np.frombuffer(bp, TPIECE, np_)
        self.vwb = np.frombuffer(bw1, "<i4", nw1)
        self.twb = np.frombuffer(bw2, "<i4", nw2)
        self.nwaves = max(len(self.vwb) - 1, 0)


class Plan:
    def __init__(self, path):
        secs = _read(path)
        hdr = np.frombuffer(secs[0][2], "<i8", 8)
        (self.pool_total, self.n_slots, self.logd_off, self.z_off, self.zw, self.n, self.n_leaves,
         self.z_slot) = map(int, hdr)
        assert secs[1][1] == DGEN.itemsize and secs[2][1] == ACA.itemsize
        self.dgen = np.frombuffer(secs[1][2], DGEN, secs[1][0])
        self.aca = np.frombuffer(secs[2][2], ACA, secs[2][0])
        self.phases = [Phase(secs[3 + 9 * i: 12 + 9 * i]) for i in range(4)]
        self.recompress, self.chol, self.solve, self.lmul = self.phases


class Interp:
    """mode "waves": tasks of each wave in random order, waves in sequence (the
    launch-per-wave executor).  mode "dag": a random topological order that
    respects only the explicit dependency lists xt/xdeps (what the persistent
    executor k_exec enforces) -- a missing edge shows up as a wrong answer."""

    def __init__(self, plan: Plan, eps: float, seed: int = 0, mode: str = "waves", rel_eps: bool = False):
        self.mode = mode
        self.rel_eps = rel_eps
        self.P = plan
        self.eps = eps
        self.pool = np.zeros(plan.pool_total)
        self.ranks = np.zeros(max(plan.n_slots, 1), dtype=np.int64)
        self.rng = np.random.default_rng(seed)
        self.fail = 0

    # ---------------------------------------------------------------- helpers
    def dim(self, d):
        if d["slot"] < 0:
            return int(d["stat"])
        v = int(self.ranks[d["slot"]]) - int(d["off"])
        return max(0, min(v, int(d["stat"])))

    def gload(self, off, ld, r, c):
        if r == 0 or c == 0:
            return np.zeros((r, c))
        idx = off + np.arange(r)[:, None] + ld * np.arange(c)[None, :]
        return self.pool[idx]

    def gstore(self, off, ld, M):
        r, c = M.shape
        if r == 0 or c == 0:
            return
        idx = off + np.arange(r)[:, None] + ld * np.arange(c)[None, :]
        self.pool[idx] = M

    # ---------------------------------------------------------------- assembly (oracle entries)
    def cut(self, smax):
        """Truncation threshold: absolute eps * sigma^2 (device default, Remark 2) or
        relative eps * sigma_1 (rel_eps)."""
        return self.eps * smax if self.rel_eps else self.eps * self.sigma2

    def assemble(self, pts_tree, theta):
        s2, ell, nu = theta
        self.sigma2 = float(s2)

        def block(r0, c0, m, q):
            a = pts_tree[r0:r0 + m]
            b = pts_tree[c0:c0 + q]
            h = np.sqrt(((a[:, None, :] - b[None, :, :]) ** 2).sum(-1))
            return matern(h.ravel(), s2, ell, nu).reshape(m, q)

        for t in self.P.dgen:
            self.gstore(int(t["off"]), int(t["m"]), block(int(t["r0"]), int(t["c0"]), int(t["m"]), int(t["q"])))
        for t in self.P.aca:
            M = block(int(t["r0"]), int(t["c0"]), int(t["m"]), int(t["q"]))
            U, S, Vt = np.linalg.svd(M, full_matrices=False)
            r = int(np.sum(S > 0.25 * self.cut(S[0]))) if S.size else 0
            r = min(r, int(t["cap"]))
            self.gstore(int(t["u_off"]), int(t["m"]), U[:, :r] * S[:r])
            self.gstore(int(t["v_off"]), int(t["q"]), Vt[:r].T)
            self.ranks[t["rslot"]] = r
        self.run(self.P.recompress)

    # ---------------------------------------------------------------- tasks
    def vm(self, ph, task):
        tiles = [np.zeros((0, 0)) for _ in range(5)]
        for I in ph.ins[task["ins_begin"]: task["ins_begin"] + task["ins_count"]]:
            op = int(I["op"])
            if op == VM_LD:
                tiles[I["t0"]] = self.gload(int(I["goff"]), int(I["ld"]), self.dim(I["rows"]), self.dim(I["cols"]))
            elif op == VM_ST:
                T = tiles[I["t0"]]
                r, c = min(self.dim(I["rows"]), T.shape[0]), min(self.dim(I["cols"]), T.shape[1])
                self.gstore(int(I["goff"]), int(I["ld"]), T[:r, :c])
            elif op == VM_ZERO:
                tiles[I["t0"]] = np.zeros((self.dim(I["rows"]), self.dim(I["cols"])))
            elif op == VM_GEMM:
                A = tiles[I["t1"]].T if I["ta"] else tiles[I["t1"]]
                B = tiles[I["t2"]].T if I["tb"] else tiles[I["t2"]]
                k = max(A.shape[1], B.shape[0])
                A2 = np.zeros((A.shape[0], k)); A2[:, :A.shape[1]] = A
                B2 = np.zeros((k, B.shape[1])); B2[:B.shape[0], :] = B
                prod = I["alpha"] * (A2 @ B2)
                if I["beta"] == 0.0:
                    tiles[I["t0"]] = prod
                else:
                    C = tiles[I["t0"]].copy()
                    C[:prod.shape[0], :prod.shape[1]] = I["beta"] * C[:prod.shape[0], :prod.shape[1]] + prod
                    tiles[I["t0"]] = C
            elif op == VM_MGEMM_ST:       # pool[dst] = beta pool[dst] + sum alpha op(A) op(B)
                r, c = self.dim(I["rows"]), self.dim(I["cols"])
                C = self.gload(int(I["goff"]), int(I["ld"]), r, c) * float(I["beta"])
                for tm in ph.terms[int(I["p2"]): int(I["p2"]) + int(I["t1"])]:
                    A = self.gload(int(tm["a_off"]), int(tm["a_ld"]), self.dim(tm["a_rows"]), self.dim(tm["a_cols"]))
                    B = self.gload(int(tm["b_off"]), int(tm["b_ld"]), self.dim(tm["b_rows"]), self.dim(tm["b_cols"]))
                    A = A.T if tm["ta"] else A
                    B = B.T if tm["tb"] else B
                    k = min(A.shape[1], B.shape[0])
                    prod = tm["alpha"] * (A[:, :k] @ B[:k, :])
                    rr, cc = min(r, prod.shape[0]), min(c, prod.shape[1])
                    C[:rr, :cc] += prod[:rr, :cc]
                self.gstore(int(I["goff"]), int(I["ld"]), C)
            elif op == VM_ADD:            # t0 += t1 (same logical dims)
                A = tiles[I["t0"]].copy()
                B = tiles[I["t1"]]
                A[:B.shape[0], :B.shape[1]] += B
                tiles[I["t0"]] = A
            elif op == VM_TRTRI:          # t0 <- inverse of the lower-triangular t1
                Lt = np.tril(tiles[I["t1"]])
                tiles[I["t0"]] = np.linalg.solve(Lt, np.eye(Lt.shape[0])) if Lt.size else Lt.copy()
            elif op == VM_MGEMM:          # t0 += sum alpha op(A) op(B), operands straight from the pool
                C = tiles[I["t0"]].copy()
                for tm in ph.terms[int(I["goff"]): int(I["goff"]) + int(I["ld"])]:
                    A = self.gload(int(tm["a_off"]), int(tm["a_ld"]), self.dim(tm["a_rows"]), self.dim(tm["a_cols"]))
                    B = self.gload(int(tm["b_off"]), int(tm["b_ld"]), self.dim(tm["b_rows"]), self.dim(tm["b_cols"]))
                    A = A.T if tm["ta"] else A
                    B = B.T if tm["tb"] else B
                    k = min(A.shape[1], B.shape[0])
                    prod = tm["alpha"] * (A[:, :k] @ B[:k, :])
                    C[:prod.shape[0], :prod.shape[1]] += prod
                tiles[I["t0"]] = C
            elif op == VM_POTRF:
                A = tiles[I["t0"]]
                A = np.tril(A) + np.tril(A, -1).T
                try:
                    L = np.linalg.cholesky(A)
                except np.linalg.LinAlgError:
                    self.fail += 1
                    L = np.eye(A.shape[0])
                tiles[I["t0"]] = L
                self.pool[int(I["goff"])] = float(np.sum(np.log(np.diag(L))))
            elif op == VM_TRSM_RLT:       # B <- B L^{-T}
                B, L = tiles[I["t0"]], tiles[I["t1"]][:tiles[I["t0"]].shape[1], :tiles[I["t0"]].shape[1]]
                tiles[I["t0"]] = np.linalg.solve(np.tril(L), B.T).T
            elif op == VM_TRSM_LN:        # B <- L^{-1} B
                B = tiles[I["t0"]]
                L = np.tril(tiles[I["t1"]][:B.shape[0], :B.shape[0]])
                tiles[I["t0"]] = np.linalg.solve(L, B)
            elif op == VM_TRMM_LN:
                B = tiles[I["t0"]]
                L = np.tril(tiles[I["t1"]][:B.shape[0], :B.shape[0]])
                tiles[I["t0"]] = L @ B
            else:
                raise ValueError(op)

    def run_trunc(self, ph, t):
        """A truncation at its share eps_scale of the block accuracy (split truncations)."""
        e = self.eps
        self.eps = e * float(t["eps_scale"])
        try:
            self.trunc(ph, t)
        finally:
            self.eps = e

    def trunc(self, ph, t):
        m, q = int(t["m"]), int(t["q"])
        As, Bs = [], []
        for pc in ph.tp[t["piece_begin"]: t["piece_begin"] + t["piece_count"]]:
            w = self.dim(pc["w"])
            A = np.zeros((m, w)); B = np.zeros((q, w))
            A[pc["u_row0"]:pc["u_row0"] + pc["u_rows"]] = pc["alpha"] * self.gload(int(pc["u_off"]), int(pc["u_ld"]),
                                                                                  int(pc["u_rows"]), w)
            B[pc["v_row0"]:pc["v_row0"] + pc["v_rows"]] = self.gload(int(pc["v_off"]), int(pc["v_ld"]),
                                                                     int(pc["v_rows"]), w)
            As.append(A); Bs.append(B)
        A = np.concatenate(As, axis=1); B = np.concatenate(Bs, axis=1)
        if A.shape[1] == 0:
            self.ranks[t["rslot"]] = 0
            return
        Qa, Ra = np.linalg.qr(A)
        Qb, Rb = np.linalg.qr(B)
        W, S, Zt = np.linalg.svd(Ra @ Rb.T)
        r = int(np.sum((S > self.cut(S[0])) & (S > 0))) if S.size else 0
        r = min(r, int(t["cap"]))
        self.gstore(int(t["u_out"]), m, (Qa @ W[:, :r]) * S[:r])
        self.gstore(int(t["v_out"]), q, Qb @ Zt[:r].T)
        self.ranks[t["rslot"]] = r

    def run(self, ph):
        if self.mode == "dag":
            return self.run_dag(ph)
        for w in range(ph.nwaves):
            jobs = [("v", i) for i in range(ph.vwb[w], ph.vwb[w + 1])] + \
                   [("t", i) for i in range(ph.twb[w], ph.twb[w + 1])]
            for kind, i in [jobs[j] for j in self.rng.permutation(len(jobs))]:
                if kind == "v":
                    self.vm(ph, ph.vt[i])
                else:
                    self.run_trunc(ph, ph.tt[i])

    def run_dag(self, ph):
        n = len(ph.xt)
        succ = [[] for _ in range(n)]
        indeg = np.zeros(n, dtype=np.int64)
        for i, x in enumerate(ph.xt):
            for d in ph.xdeps[x["dep_begin"]: x["dep_begin"] + x["dep_count"]]:
                assert d < i, "dependency must precede the task in xt order"
                succ[int(d)].append(i)
                indeg[i] += 1
        ready = [i for i in range(n) if indeg[i] == 0]
        done = 0
        while ready:
            j = int(self.rng.integers(len(ready)))
            i = ready[j]
            ready[j] = ready[-1]
            ready.pop()
            x = ph.xt[i]
            if x["kind"] == 0:
                self.vm(ph, ph.vt[x["idx"]])
            elif x["sub"] == 0:              # a cooperative truncation runs once (its leader)
                self.run_trunc(ph, ph.tt[x["idx"]])
            done += 1
            for s2 in succ[i]:
                indeg[s2] -= 1
                if indeg[s2] == 0:
                    ready.append(s2)
        assert done == n

    # ---------------------------------------------------------------- likelihood
    def loglik(self, Z_tree):
        n, zw = self.P.n, self.P.zw
        Z_tree = np.asarray(Z_tree).reshape(n, -1)
        k = Z_tree.shape[1]
        buf = np.zeros((n, zw))
        buf[:, :k] = Z_tree
        self.pool[self.P.z_off:self.P.z_off + n * zw] = buf.ravel(order="F")
        self.ranks[self.P.z_slot] = k            # active columns of the z buffer (hm_loglik)
        self.run(self.P.solve)
        v = self.pool[self.P.z_off:self.P.z_off + n * zw].reshape(zw, n).T[:, :k]
        logdet = 2.0 * float(np.sum(self.pool[self.P.logd_off:self.P.logd_off + self.P.n_leaves]))
        quad = np.sum(v * v, axis=0)
        return -0.5 * n * math.log(2 * math.pi) - 0.5 * logdet - 0.5 * quad, logdet, quad

    def lmul(self, X_tree):
        n, zw = self.P.n, self.P.zw
        X_tree = np.asarray(X_tree).reshape(n, -1)
        k = X_tree.shape[1]
        buf = np.zeros((n, zw))
        buf[:, :k] = X_tree
        self.pool[self.P.z_off:self.P.z_off + n * zw] = buf.ravel(order="F")
        self.ranks[self.P.z_slot] = k
        self.run(self.P.lmul)
        return self.pool[self.P.z_off:self.P.z_off + n * zw].reshape(zw, n).T[:, :k].copy()


class InterpRand(Interp):
    """Interp whose wide truncations follow the device's randomized range finder
    (trunc.cuh, trunc_rand) step by step: rounds of RB Gaussian probes, block
    Gram-Schmidt twice (BCGS2) with a pivoted Cholesky-QR of each block (pivots
    above max(eps * max_j ||M w_j||, 1e-4 * largest)) and a CholQR of the
    re-projected block, stopping when the largest projected probe is below
    eps * max_j ||M w_j|| (relative Frobenius certificate), then
    W = M^T Q, QR, SVD of R^T,
    U = Q X', V = W X' Sigma^-2.  Used to check that algorithm on the CPU."""
    RB = 8             # hm_tasks.h TR_RB
    EXACT_K = 160      # hm_tasks.h TR_EXACT_K / TR_EXACT_MMAX (trunc_exact_path)
    EXACT_MMAX = 512

    def trunc(self, ph, t):
        if int(t["kmax_tot"]) <= self.EXACT_K and int(t["m"]) <= self.EXACT_MMAX and int(t["q"]) <= self.EXACT_MMAX:
            return super().trunc(ph, t)
        m, q, cap = int(t["m"]), int(t["q"]), int(t["cap"])
        As, Bs = [], []
        for pc in ph.tp[t["piece_begin"]: t["piece_begin"] + t["piece_count"]]:
            w = self.dim(pc["w"])
            A = np.zeros((m, w)); B = np.zeros((q, w))
            A[pc["u_row0"]:pc["u_row0"] + pc["u_rows"]] = pc["alpha"] * self.gload(int(pc["u_off"]), int(pc["u_ld"]),
                                                                                  int(pc["u_rows"]), w)
            B[pc["v_row0"]:pc["v_row0"] + pc["v_rows"]] = self.gload(int(pc["v_off"]), int(pc["v_ld"]),
                                                                     int(pc["v_rows"]), w)
            As.append(A); Bs.append(B)
        A = np.concatenate(As, axis=1); B = np.concatenate(Bs, axis=1)
        L = cap + self.RB
        Q = np.zeros((m, 0))
        sest = 0.0
        while True:
            Om = self.rng.standard_normal((q, self.RB))
            Y = A @ (B.T @ Om)
            sest = max(sest, float(np.max(np.linalg.norm(Y, axis=0))))   # ~ ||M||_F
            thr = (self.eps * sest if self.rel_eps else self.eps * self.sigma2) * 1.0   # TR_STOP
            for _ in range(2):                       # BCGS2, first projection (twice)
                Y = Y - Q @ (Q.T @ Y)
            G = Y.T @ Y                              # pivoted Cholesky-QR of the block
            d0 = float(np.max(np.diag(G)))
            maxn = math.sqrt(max(d0, 0.0))
            cut = max(thr * thr, 1e-8 * d0)
            piv = list(range(self.RB))
            R = np.zeros((self.RB, self.RB))
            na = 0
            for k in range(self.RB):
                if Q.shape[1] + k >= L:
                    break
                jb = k + int(np.argmax([G[piv[j], piv[j]] for j in range(k, self.RB)]))
                piv[k], piv[jb] = piv[jb], piv[k]
                d = G[piv[k], piv[k]]
                if not d > cut:
                    break
                R[k, k] = math.sqrt(d)
                for j in range(k + 1, self.RB):
                    R[k, j] = G[piv[k], piv[j]] / R[k, k]
                for i in range(k + 1, self.RB):
                    for j in range(i, self.RB):
                        v = G[piv[i], piv[j]] - R[k, i] * R[k, j]
                        G[piv[i], piv[j]] = v
                        G[piv[j], piv[i]] = v
                na += 1
            added = []
            if na:
                Qn = scipy.linalg.solve_triangular(R[:na, :na], Y[:, piv[:na]].T, trans="T", lower=False).T
                Qn = Qn - Q @ (Q.T @ Qn)             # second projection of the new block
                R2 = np.linalg.cholesky(Qn.T @ Qn).T  # CholQR of the nearly orthonormal block
                Qn = scipy.linalg.solve_triangular(R2, Qn.T, trans="T", lower=False).T
                Q = np.concatenate([Q, Qn], axis=1)
                added = [0] * na
            if maxn <= thr or not added or Q.shape[1] >= L or Q.shape[1] >= m or Q.shape[1] >= q:
                break
        if Q.shape[1] == 0:
            self.ranks[t["rslot"]] = 0
            return
        Wm = B @ (A.T @ Q)                           # W = M^T Q
        if self.eps >= 1e-7:                         # TR_GRAM_EPS: pivoted Cholesky of W^T W
            G = Wm.T @ Wm
            ell = G.shape[0]
            cut = (self.eps ** 2 * float(np.max(np.diag(G)))) if self.rel_eps else (self.eps * self.sigma2) ** 2
            piv = list(range(ell))
            R = np.zeros((ell, ell))
            r = 0
            for k in range(ell):
                jb = k + int(np.argmax([G[piv[j], piv[j]] for j in range(k, ell)]))
                piv[k], piv[jb] = piv[jb], piv[k]
                d = G[piv[k], piv[k]]
                if not d > cut:
                    break
                if k >= cap:
                    break
                R[k, k] = math.sqrt(d)
                for j in range(k + 1, ell):
                    R[k, j] = G[piv[k], piv[j]] / R[k, k]
                for i in range(k + 1, ell):
                    for j in range(i, ell):
                        v = G[piv[i], piv[j]] - R[k, i] * R[k, j]
                        G[piv[i], piv[j]] = v
                        G[piv[j], piv[i]] = v
                r = k + 1
            Xo = np.zeros((ell, r))
            Gm = np.zeros((ell, r))
            Rinv = np.linalg.inv(np.triu(R[:r, :r])) if r else np.zeros((0, 0))
            for c in range(r):
                for j in range(ell):
                    if j >= c:
                        Xo[piv[j], c] = R[c, j]
                for j in range(c + 1):
                    Gm[piv[j], c] = Rinv[j, c]
            self.gstore(int(t["u_out"]), m, Q @ Xo)                # U = Q P R^T
            self.gstore(int(t["v_out"]), q, Wm @ Gm)               # V = W P_r R11^-1
            self.ranks[t["rslot"]] = r
            return
        _, R = np.linalg.qr(Wm)
        Xp, S, Zt = np.linalg.svd(R.T)               # R^T = X' Z^T with X' = Xp S
        r = int(np.sum((S > self.cut(S[0])) & (S > 0)))
        r = min(r, cap)
        Xr = Xp[:, :r] * S[:r]
        self.gstore(int(t["u_out"]), m, Q @ Xr)                  # U = Q X'
        self.gstore(int(t["v_out"]), q, Wm @ (Xr / S[:r] ** 2))   # V = W X' Sigma^-2 (= Q_W Z)
        self.ranks[t["rslot"]] = r
