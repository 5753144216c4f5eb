// Low-rank truncation kernel k_trunc ("efficient rank-truncation
// techniques"; adaptive-rank strategy of Remark 2, l.166, reading R4):
//
//   B <- best rank-r approximation, sigma_i > tau, of
//        M = sum_p alpha_p pad(U_p) pad(V_p)^T        (m x q, K = sum_p width_p)
//
// Two algorithms, chosen per task by the planner's static width bound:
//  * EXACT (static K <= TR_EXACT_K, e.g. the recompression after ACA): gather the
//    stacks A (m x K), B (q x K); Householder QR of both; one-sided Jacobi SVD of
//    the core R_A R_B^T; U = Q_A X Sigma, V = Q_B Z.
//  * RANDOMIZED (wide stacks -- an H-Cholesky block gathers one piece per
//    product of its block row, K reaches thousands): adaptive randomized range
//    finder on the implicit sum (Halko, Martinsson & Tropp, Alg. 4.2 with the
//    a-posteriori bound of their Lemma 4.1): rounds of RB Gaussian probes
//    Y = M Omega computed piece by piece (never forming M or the stacks),
//    twice-projected against the basis Q, stop when every projected probe of a
//    round has norm <= TR_STOP * tau (an estimate of ||M - Q Q^T M||_F, which
//    bounds the spectral error); then W = M^T Q (again piece by piece),
//    Householder QR W = Q_W R, Jacobi SVD of R^T, U = Q X Sigma, V = Q_W Z.
//    Work is linear in K (about 4 (m + q) K (ell + RB) flops), and the only
//    dense SVD is ell x ell with ell = rank + RB.
// One CTA per task (k_trunc: all tasks of a wave in one launch; k_exec: claimed
// one at a time by persistent CTAs).

// dispatch on the planner's static width bound

#pragma once
#include <cuda_runtime.h>

#include <cfloat>
#include <cmath>
#include <cstdint>

#include "dev_util.cuh"
#include "hm_kernels.h"
#include "hm_tasks.h"
#include "gemm.cuh"
#include "tile.cuh"

namespace hm {

constexpr int TR_THREADS = 256;

// truncation threshold tau: eps > 0 relative (sigma_i > eps sigma_1), eps < 0 absolute
// (sigma_i > |eps| = eps * sigma^2, the default: the paper's Remark 2 wording, reading R4)
__device__ __forceinline__ double tr_cut(double eps, double smax) { return eps > 0.0 ? eps * smax : -eps; }
constexpr int ORDER_MAX = 512;
// exact path in shared memory: behind `order` (ORDER_MAX ints), up to TR_XS_DOUBLES doubles
constexpr int TR_XS_OFF = ORDER_MAX / 2;
constexpr int TR_XS_DOUBLES = 22016;              // 172 KB: e.g. 256 + 256 rows x K = 36
// Range-finder stopping rule.  For a Gaussian probe w, E ||R w||^2 = ||R||_F^2, so
// the probe norms ||M w_j|| estimate ||M||_F and the projected-probe norms
// ||(I - Q Q^T) M w_j|| estimate ||M - Q Q^T M||_F.  The basis is complete when
// every projected probe of a round is <= TR_STOP * tau (tau = the truncation threshold,
// |eps| absolute or eps * max_j ||M w_j|| relative): Frobenius accuracy ~TR_STOP * tau,
// hence also spectral, before the final SVD truncation at tau.  TR_STOP = 1 certifies
// Remark 2's "accuracy eps or better" per block (l.166-167); the round-1 value 4 kept
// the noise floor of the accumulated updates (bases ~40 % narrower) at ~4 tau.
#ifndef HM_TR_STOP
#define HM_TR_STOP 1.0
#endif
constexpr double TR_STOP = HM_TR_STOP;
// eps from which the final SVD of the projected block uses the Gram matrix (see F3)
constexpr double TR_GRAM_EPS = 1e-7;

// dynamic shared memory: [Cs (leader) | staging] then order, koff
constexpr int TR_SMEM_A = 8 * GEMM_SMEM_DOUBLES;   // GEMM staging, then order / koff

// Householder QR of A (m x K, ld m) in place; tau[K].  R in the upper triangle, the
// reflectors v (v_i = 1 implicit) below it.  Two CTA barriers per column: the
// reflector is applied in its unscaled form (the scale 1 / (alpha - beta) folded
// into w), the warp that updates column i + 1 also forms that column's norm below
// the diagonal for the next step, and the reflectors are scaled in one pass at the end.
// sc: K doubles of scratch (shared memory preferred).
static __device__ __noinline__ void house_qr(double* A, int m, int K, double* tau, double* sc) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int kmin = min(m, K);
    __shared__ double s_sig, s_tau, s_sc;
    if (warp == 0) {                                   // norm of column 0 below the diagonal
        double ss = 0.0;
        for (int r = 1 + lane; r < m; r += 32) ss += A[r] * A[r];
        ss = warp_sum(ss);
        if (lane == 0) s_sig = ss;
    }
    __syncthreads();
    for (int i = 0; i < kmin; ++i) {
        double* a = A + (int64_t)i * m;
        if (threadIdx.x == 0) {
            const double alpha = a[i], sig = s_sig;
            if (sig == 0.0) {
                s_tau = 0.0;
                s_sc = 0.0;
            } else {
                const double nrm = sqrt(alpha * alpha + sig);
                const double beta = (alpha <= 0.0) ? nrm : -nrm;
                s_tau = (beta - alpha) / beta;
                s_sc = 1.0 / (alpha - beta);
                a[i] = beta;
            }
            tau[i] = s_tau;
            sc[i] = s_sc;
            s_sig = 0.0;
        }
        __syncthreads();
        const double tv = s_tau, scl = s_sc;
        // apply H = I - tau v v^T (v_i = 1, v_r = scl a_r) to columns c > i: one warp per column
        for (int c = i + 1 + warp; c < K; c += nw) {
            double* col = A + (int64_t)c * m;
            if (tv != 0.0) {
                double w = 0.0;
                for (int r = i + 1 + lane; r < m; r += 32) w += a[r] * col[r];
                w = (warp_sum(w) * scl + col[i]) * tv;
                if (lane == 0) col[i] -= w;
                const double ws = w * scl;
                for (int r = i + 1 + lane; r < m; r += 32) col[r] -= ws * a[r];
            }
            if (c == i + 1) {                          // next column's norm below its diagonal
                __syncwarp();
                double ss = 0.0;
                for (int r = i + 2 + lane; r < m; r += 32) ss += col[r] * col[r];
                ss = warp_sum(ss);
                if (lane == 0) s_sig = ss;
            }
        }
        __syncthreads();
    }
    for (int i = warp; i < kmin; i += nw) {            // scale the reflectors
        double* a = A + (int64_t)i * m;
        const double scl = sc[i];
        for (int r = i + 1 + lane; r < m; r += 32) a[r] *= scl;
    }
    __syncthreads();
}

// Y (m x r, ld m) <- Q Y with Q = H_0 H_1 ... H_{kmin-1} stored in A (m x K) / tau
static __device__ __noinline__ void house_apply_q(const double* A, int m, int kmin, const double* tau, double* Y, int r) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int i = kmin - 1; i >= 0; --i) {
        const double tv = tau[i];
        if (tv == 0.0) continue;
        const double* a = A + (int64_t)i * m;
        for (int c = warp; c < r; c += nw) {
            double* col = Y + (int64_t)c * m;
            double w = (lane == 0) ? col[i] : 0.0;
            for (int rr = i + 1 + lane; rr < m; rr += 32) w += a[rr] * col[rr];
            w = warp_sum(w) * tv;
            if (lane == 0) col[i] -= w;
            for (int rr = i + 1 + lane; rr < m; rr += 32) col[rr] -= w * a[rr];
        }
        __syncthreads();
    }
}

// one-sided Jacobi: X (rows x n, ld rows) -> X Z with orthogonal columns; Z (n x n, ld n).
// Round-robin pairing, one pair per half-warp (16 lanes stride the rows), so a round of
// up to 16 pairs is one pass of the 8 warps; the half-warp sums use 4 shuffle levels.
__device__ __forceinline__ double half_sum(double v) {
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
static __device__ __noinline__ void jacobi_svd(double* X, int rows, int n, double* Z, int* s_flag) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int hl = lane & 15, half = lane >> 4;
    for (int idx = threadIdx.x; idx < n * n; idx += blockDim.x) Z[idx] = ((idx % n) == (idx / n)) ? 1.0 : 0.0;
    __syncthreads();
    if (n < 2) return;
    const int nn = (n + 1) & ~1;   // even number of players (one dummy if n odd)
    for (int sweep = 0; sweep < 16; ++sweep) {
        if (threadIdx.x == 0) *s_flag = 0;
        __syncthreads();
        for (int round = 0; round < nn - 1; ++round) {
            // all lanes of a warp take the same number of steps (the shuffles need both halves)
            for (int base = 2 * warp; base < nn / 2; base += 2 * nw) {
                const int pr = base + half;
                // round-robin pairing: player 0 fixed, others rotate
                int a = (pr == 0) ? 0 : ((round + pr - 1) % (nn - 1)) + 1;
                int b = ((round + nn - 2 - pr) % (nn - 1)) + 1;
                if (pr == 0) b = ((round + nn - 2) % (nn - 1)) + 1;
                const bool act = pr < nn / 2 && a < n && b < n;
                if (a > b) { int tmp = a; a = b; b = tmp; }
                double* xa = X + (int64_t)(act ? a : 0) * rows;
                double* xb = X + (int64_t)(act ? b : 0) * rows;
                double al = 0.0, be = 0.0, ga = 0.0;
                if (act)
                    for (int r = hl; r < rows; r += 16) {
                        const double u = xa[r], v = xb[r];
                        al += u * u; be += v * v; ga += u * v;
                    }
                al = half_sum(al); be = half_sum(be); ga = half_sum(ga);
                if (act && fabs(ga) > 1e-14 * sqrt(al * be) && ga != 0.0) {
                    const double zeta = (be - al) / (2.0 * ga);
                    const double tt = ((zeta >= 0.0) ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                    const double c = 1.0 / sqrt(1.0 + tt * tt), s = c * tt;
                    for (int r = hl; r < rows; r += 16) {
                        const double u = xa[r], v = xb[r];
                        xa[r] = c * u - s * v;
                        xb[r] = s * u + c * v;
                    }
                    double* za = Z + (int64_t)a * n;
                    double* zb = Z + (int64_t)b * n;
                    for (int r = hl; r < n; r += 16) {
                        const double u = za[r], v = zb[r];
                        za[r] = c * u - s * v;
                        zb[r] = s * u + c * v;
                    }
                    if (hl == 0) *s_flag = 1;
                }
            }
            __syncthreads();
        }
        if (*s_flag == 0) break;
        __syncthreads();
    }
    __syncthreads();
}


// jacobi_svd with X (rows x n) and Z (n x n) staged in shared memory when they fit the
// GEMM staging area (the small SVD is latency-bound; global memory makes it ~10x slower)
static __device__ __forceinline__ void jacobi_smem(double* X, int rows, int n, double* Z, double* sm, int* s_flag) {
    if ((int64_t)rows * n + (int64_t)n * n <= GEMM_SMEM_DOUBLES) {
        double* Xs = sm;
        double* Zs = sm + rows * n;
        for (int i = threadIdx.x; i < rows * n; i += blockDim.x) Xs[i] = X[i];
        __syncthreads();
        jacobi_svd(Xs, rows, n, Zs, s_flag);
        for (int i = threadIdx.x; i < rows * n; i += blockDim.x) X[i] = Xs[i];
        for (int i = threadIdx.x; i < n * n; i += blockDim.x) Z[i] = Zs[i];
        __syncthreads();
    } else {
        jacobi_svd(X, rows, n, Z, s_flag);
    }
}

// ---------------------------------------------------------------- exact path
// dst (len x w, ld len) = al * rows [row0, row0 + rows) of the piece src (ld sld), zero
// elsewhere.  The element loop is batched 8 deep (all loads, then all stores): one
// load in flight per thread made the gathers latency-bound.  Pieces are written by
// other CTAs of the persistent executor: read through L2.
__device__ __forceinline__ void gather_cols(double* __restrict__ dst, int len, const double* __restrict__ src,
                                            int64_t sld, int row0, int rows, int w, double al) {
    const int tot = len * w;                       // exact path: len <= TR_EXACT_MMAX, w <= K
    for (int base = threadIdx.x; base < tot; base += 8 * blockDim.x) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int idx = base + u * blockDim.x;
            v[u] = 0.0;
            if (idx < tot) {
                const int r = idx % len, c = idx / len;
                const int rr = r - row0;
                if (rr >= 0 && rr < rows) v[u] = al * __ldcg(src + rr + (int64_t)c * sld);
            }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int idx = base + u * blockDim.x;
            if (idx < tot) dst[idx] = v[u];
        }
    }
}

static __device__ void trunc_exact(const TTask& t, int K, const TPiece* __restrict__ pieces, double* __restrict__ pool,
                            int* __restrict__ ranks, int* __restrict__ flags, double eps, double* __restrict__ ctr,
                            double* dsm) {
    __shared__ double scratch[32];
    __shared__ double s_hsc[TR_EXACT_K];           // Householder scales
    int* order = (int*)dsm;                        // ORDER_MAX ints (dynamic shared memory)
    __shared__ int s_flag;
    __shared__ int s_rank;
    const int m = t.m, q = t.q;
    // the stacks, cores and factors live in shared memory when they fit (the column-serial
    // QR and the Jacobi sweeps are latency-bound: global memory made them several times
    // slower), else in the task's global workspace
    const bool insm = (int64_t)(m + q + 3) * K + 2 * (int64_t)K * K <= TR_XS_DOUBLES;
    double* ws = insm ? dsm + TR_XS_OFF : pool + t.ws;
    double* A = ws;                       // m x K
    double* Bm = A + (int64_t)m * K;      // q x K
    double* tauA = Bm + (int64_t)q * K;   // K
    double* tauB = tauA + K;              // K
    double* sig = tauB + K;               // K
    double* X = sig + K;                  // Ka x Kb  (<= K x K)
    double* Z = X + (int64_t)K * K;       // Kb x Kb
    // gather
    int koff = 0;
    for (int pi = 0; pi < t.piece_count; ++pi) {
        const TPiece pc = pieces[t.piece_begin + pi];
        const int w = dim_eval(pc.w, ranks);
        const double* Up = pool + pc.u_off;
        const double* Vp = pool + pc.v_off;
        gather_cols(A + (int64_t)koff * m, m, Up, pc.u_ld, pc.u_row0, pc.u_rows, w, pc.alpha);
        gather_cols(Bm + (int64_t)koff * q, q, Vp, pc.v_ld, pc.v_row0, pc.v_rows, w, 1.0);
        koff += w;
    }
    __syncthreads();
    if (K == 0) {
        if (threadIdx.x == 0) ranks[t.rslot] = 0;
        return;
    }
    house_qr(A, m, K, tauA, s_hsc);
    house_qr(Bm, q, K, tauB, s_hsc);
    const int Ka = min(m, K), Kb = min(q, K);
    // X = R_A R_B^T  (Ka x Kb), R_A[i][c] (c >= i) = A[i + c m], R_B[j][c] = Bm[j + c q]
    for (int idx = threadIdx.x; idx < Ka * Kb; idx += blockDim.x) {
        const int i = idx % Ka, j = idx / Ka;
        double s = 0.0;
        for (int c = max(i, j); c < K; ++c) s += A[i + (int64_t)c * m] * Bm[j + (int64_t)c * q];
        X[i + (int64_t)j * Ka] = s;
    }
    __syncthreads();
    // the small SVD is latency-bound: staged in shared memory behind `order` when it fits
    // (Ka x Kb + Kb x Kb doubles, i.e. K <= 68; global memory made it ~10x slower)
    if (insm) jacobi_svd(X, Ka, Kb, Z, &s_flag);
    else jacobi_smem(X, Ka, Kb, Z, dsm + ORDER_MAX / 2, &s_flag);
    // singular values = column norms of X
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int j = warp; j < Kb; j += nw) {
        double s = 0.0;
        for (int r = lane; r < Ka; r += 32) s += X[r + (int64_t)j * Ka] * X[r + (int64_t)j * Ka];
        s = warp_sum(s);
        if (lane == 0) sig[j] = sqrt(s);
    }
    __syncthreads();
    // order by decreasing sigma (rank counting, ties by index), rank by eps * sigma_max
    __shared__ double s_smax;
    const int kk = min(Kb, ORDER_MAX);
    for (int j = threadIdx.x; j < kk; j += blockDim.x) {
        int pos = 0;
        const double sj = sig[j];
        for (int b = 0; b < kk; ++b) pos += (sig[b] > sj || (sig[b] == sj && b < j)) ? 1 : 0;
        order[pos] = j;
    }
    __syncthreads();
    if (threadIdx.x == 0) s_smax = (kk > 0) ? sig[order[0]] : 0.0;
    __syncthreads();
    {
        int cnt = 0;
        for (int j = threadIdx.x; j < kk; j += blockDim.x) cnt += (sig[j] > tr_cut(eps, s_smax) && sig[j] > 0.0) ? 1 : 0;
        const double tot = block_sum((double)cnt, scratch);
        if (threadIdx.x == 0) {
            int r = (int)(tot + 0.5);
            if (r > t.cap) { atomicOr(flags + 1, 2); r = t.cap; }
            s_rank = r;
        }
    }
    __syncthreads();
    const int r = s_rank;
    // U_out = Q_A [X(:, order) ; 0],  V_out = Q_B [Z(:, order) ; 0]
    double* Uo = pool + t.u_out;
    double* Vo = pool + t.v_out;
    for (int idx = threadIdx.x; idx < m * r; idx += blockDim.x) {
        const int i = idx % m, c = idx / m;
        Uo[i + (int64_t)c * m] = (i < Ka) ? X[i + (int64_t)order[c] * Ka] : 0.0;
    }
    for (int idx = threadIdx.x; idx < q * r; idx += blockDim.x) {
        const int i = idx % q, c = idx / q;
        Vo[i + (int64_t)c * q] = (i < Kb) ? Z[i + (int64_t)order[c] * Kb] : 0.0;
    }
    __syncthreads();
    house_apply_q(A, m, Ka, tauA, Uo, r);
    house_apply_q(Bm, q, Kb, tauB, Vo, r);
    if (threadIdx.x == 0) {
        ranks[t.rslot] = r;
        // algorithmic work: Householder QR of the m x K and q x K
        // stacks (Ka = min(m, K), Kb = min(q, K) reflectors), the Ka x Kb core R_A R_B^T, one Jacobi sweep-equivalent per column
        // pair (counted as one sweep: 6 (Ka + Kb) per pair), and Q_A, Q_B applied
        // to the r kept columns; bytes: the K (m + q) piece entries read and the
        // r (m + q) factor entries written.
        const double Kd = K, md = m, qd = q, ka = Ka, kb = Kb, rd = r;
        const double fl = 2.0 * (md * Kd * ka - ka * ka * ka / 3.0) + 2.0 * (qd * Kd * kb - kb * kb * kb / 3.0) +
                          2.0 * ka * kb * Kd / 3.0 + 3.0 * kb * (kb - 1.0) * (ka + kb) +
                          4.0 * md * ka * rd + 4.0 * qd * kb * rd;
        atomicAdd(ctr + CTR_TRUNC + 0, fl);
        atomicAdd(ctr + CTR_TRUNC + 1, 8.0 * (Kd * (md + qd) + rd * (md + qd)));
    }
}


// ---------------------------------------------------------------- randomized path
// Standard normal from a counter (splitmix64 hash -> two uniforms -> Box-Muller in
// fp32; the probe matrix needs no precision, only independence).
__device__ __forceinline__ double rnd_normal(uint64_t key) {
    uint64_t z = key + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    const float u1 = ((uint32_t)(z >> 40) + 0.5f) * (1.0f / 16777216.0f);
    const float u2 = ((uint32_t)(z & 0xFFFFFFu) + 0.5f) * (1.0f / 16777216.0f);
    return (double)(sqrtf(-2.0f * __logf(u1)) * __cosf(6.2831853f * u2));
}

// acc[j] (j < RB) warp-reduced; lane 0 ends with the totals
__device__ __forceinline__ void warp_sum_arr(double* acc) {
#pragma unroll
    for (int j = 0; j < TR_RB; ++j) acc[j] = warp_sum(acc[j]);
}


// Barrier among the nsub CTAs of one cooperative truncation (persistent executor
// only: the nsub sub-tasks are consecutive in the claim order, nsub <= grid).
__device__ __forceinline__ void coop_sync(int* bar, int nsub, int& gen, unsigned long long* st = nullptr) {
    if (st && threadIdx.x == 0 && gen < 60) {   // stage timestamps (diagnostics, hm_trace)
        unsigned long long now;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
        st[gen + 1] = now;
    }
    __syncthreads();
    ++gen;
    if (nsub > 1) {
        if (threadIdx.x == 0) {
            __threadfence();
            atomicAdd(bar, 1);
            const int target = gen * nsub;
            // Liveness rests on the group's CTAs being co-resident (exec.cu); a partner
            // that never arrives (e.g. other work holding the SMs) traps after
            // TR_COOP_WATCHDOG_NS instead of hanging: the launch fails, hm_* -> HM_ERR_CUDA.
            const unsigned long long t0 = gtimer();
            while (ld_acquire_gpu(bar) < target) {
                __nanosleep(32);
                if (gtimer() - t0 > TR_COOP_WATCHDOG_NS) __trap();
            }
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
        }
        __syncthreads();
    }
}

// C (M x N, ldc) = op(A) op(B) with the inner dimension Kd cut into rs parts when the output
// has fewer tiles (64 x 64) than the group has CTAs: units (part, tile) are spread over the
// group, partials go to Rp (rs x ldp x N, ldp >= M), and each CTA then sums the columns
// [c0, c1) it owns (the caller's slice) -- the caller synchronises before reading others'.
// A and B are given at row offset 0 of the inner dimension (A: Kd x M transposed, B: Kd x N).
__device__ __forceinline__ void gemm_tn_rsplit(int M, int N, int Kd, const double* A, int64_t lda, const double* B,
                                               int64_t ldb, double* C, int64_t ldc, double* Rp, int64_t ldp, int rs,
                                               int sub, int nsub, int c0, int c1, int* bar, int& gen,
                                               unsigned long long* stt, double* gsm) {
    const int tm = (M + 63) / 64, tn = (N + 63) / 64;
    const int Kp = ((Kd + rs - 1) / rs + 15) & ~15;
    for (int u = sub; u < rs * tm * tn; u += nsub) {
        const int p = u / (tm * tn), tile = u % (tm * tn);
        const int k0 = min(Kd, p * Kp), k1 = min(Kd, k0 + Kp);
        double* Cp = Rp + (int64_t)p * ldp * N;
        if (k1 > k0) {
            gemm_wide<true, false>(M, N, k1 - k0, 1.0, gop(A + k0, lda, true), gop(B + k0, ldb, false), 0.0, Cp, ldp, tile, tm * tn,
                      gsm);
        } else {
            const int i0 = (tile % tm) * 64, j0 = (tile / tm) * 64;
            for (int idx = threadIdx.x; idx < 64 * 64; idx += blockDim.x) {
                const int i = i0 + (idx & 63), j = j0 + (idx >> 6);
                if (i < M && j < N) Cp[i + (int64_t)j * ldp] = 0.0;
            }
        }
    }
    coop_sync(bar, nsub, gen, stt);
    for (int idx = threadIdx.x; idx < M * (c1 - c0); idx += blockDim.x) {
        const int i = idx % M, j = c0 + idx / M;
        double a = 0.0;
        for (int p = 0; p < rs; ++p) a += __ldcg(Rp + (int64_t)p * ldp * N + i + (int64_t)j * ldp);
        C[i + (int64_t)j * ldc] = a;
    }
    __syncthreads();
}

// piece containing stacked column k (koff: prefix widths, np + 1 entries)
__device__ __forceinline__ int piece_of(const int* koff, int np, int k) {
    int lo = 0, hi = np - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (koff[mid] <= k) lo = mid; else hi = mid - 1;
    }
    return lo;
}



// Row ownership in a cooperative truncation: CTA sub owns the contiguous 64-row
// chunks [nch sub / nsub, nch (sub + 1) / nsub), so each of its row-local products
// is one GEMM call (one pipeline) instead of one per chunk.
__device__ __forceinline__ void own_rows(int len, int sub, int nsub, int& r0, int& r1) {
    const int nch = (len + TR_RCH - 1) / TR_RCH;
    r0 = min(len, (int)((int64_t)nch * sub / nsub) * TR_RCH);
    r1 = min(len, (int)((int64_t)nch * (sub + 1) / nsub) * TR_RCH);
}

// X[:, 0:nc] <- X - Q[:, 0:ell] (Q^T X) on this CTA's own rows [r0, r1); the ell x nc
// product is reduced over the group through per-CTA partials (one barrier).
__device__ __forceinline__ void proj_owned(const TruncWs& W, int m, int ell, int L, double* X, int nc, int sub, int nsub,
                                           int r0, int r1, int* bar, int& gen, unsigned long long* stt, double* gsm) {
    double* Cp = W.Cp + (int64_t)sub * L * TR_RB;
    if (r1 > r0)
        gemm_narrow<true, false>(ell, nc, r1 - r0, 1.0, gop(W.Q + r0, m, true), gop(X + r0, m, false), 0.0, Cp, L, 0, 1,
                                 gsm);
    else
        for (int idx = threadIdx.x; idx < ell * nc; idx += blockDim.x) Cp[(idx % ell) + (int64_t)(idx / ell) * L] = 0.0;
    coop_sync(bar, nsub, gen, stt);
    double* Cf = W.Cf + (int64_t)sub * L * TR_RB;
    for (int idx = threadIdx.x; idx < ell * nc; idx += blockDim.x) {
        const int64_t e = (idx % ell) + (int64_t)(idx / ell) * L;
        double a = 0.0;
        for (int s2 = 0; s2 < nsub; ++s2) a += __ldcg(W.Cp + (int64_t)s2 * L * TR_RB + e);
        Cf[e] = a;
    }
    __syncthreads();
    if (r1 > r0)
        gemm_narrow<false, false>(r1 - r0, nc, ell, -1.0, gop(W.Q + r0, m, false), gop(Cf, L, false), 1.0, X + r0, m, 0,
                                  1, gsm);
    // (no barrier: the partials are re-written only after the next coop_sync, and X's
    //  own rows are touched only by this CTA)
}

// Gs (shared, nc x nc, ld TR_RB) = X[:, 0:nc]^T X[:, 0:nc], reduced over the group
__device__ __forceinline__ void gram_owned(const TruncWs& W, int m, const double* X, int nc, int sub, int nsub, int r0,
                                           int r1, int* bar, int& gen, unsigned long long* stt, double* gsm,
                                           double* Gs) {
    double* Gp = W.Gp + (int64_t)sub * TR_RB * TR_RB;
    if (r1 > r0)
        gemm_short<true, false>(nc, nc, r1 - r0, 1.0, gop(X + r0, m, true), gop(X + r0, m, false), 0.0, Gp, TR_RB, 0, 1,
                                gsm);
    else
        for (int idx = threadIdx.x; idx < nc * nc; idx += blockDim.x) Gp[(idx % nc) + (idx / nc) * TR_RB] = 0.0;
    coop_sync(bar, nsub, gen, stt);
    for (int idx = threadIdx.x; idx < TR_RB * TR_RB; idx += blockDim.x) {
        const int i = idx % TR_RB, j = idx / TR_RB;
        double a = 0.0;
        if (i < nc && j < nc)
            for (int s2 = 0; s2 < nsub; ++s2) a += __ldcg(W.Gp + (int64_t)s2 * TR_RB * TR_RB + i + j * TR_RB);
        Gs[i * TR_RB + j] = a;                     // symmetric: row/col order immaterial
    }
    __syncthreads();
}

// Gram-path truncation: column-pivoted Cholesky of the ell x ell Gram matrix G = W^T W
// (P^T G P ~ R^T R, R = [R11 R12], r x ell) stopped when the largest remaining pivot
// falls below eps^2 * max diag(G).  With Q_W = W P_r R11^-1, W ~ Q_W R P^T, so
// M ~ Q W^T = (Q P R^T) Q_W^T: writes Xo (ell x r, rows in basis order) with
// Xo[piv[j], c] = R[c][j] and Gm[piv[j], c] = (R11^-1)[j][c]; U = Q Xo, V = W Gm.
// All threads of the (leader) CTA; G is staged in shared memory when it fits.
static __device__ int gram_pchol(const double* Gg, int ell, double eps, int cap, double* Xo, double* Gm, int L, double* sm,
                          int* piv, int* flags) {
    __shared__ int s_stop;
    __shared__ double s_cut;
    const bool insm = (int64_t)ell * ell <= GEMM_SMEM_DOUBLES;
    double* A = insm ? sm : const_cast<double*>(Gg);
    if (insm) {
        for (int i = threadIdx.x; i < ell * ell; i += blockDim.x) A[i] = Gg[i];
    }
    for (int i = threadIdx.x; i < ell; i += blockDim.x) piv[i] = i;
    __syncthreads();
    if (threadIdx.x == 0) {
        double d0 = 0.0;
        for (int i = 0; i < ell; ++i) d0 = fmax(d0, A[i * ell + i]);
        s_cut = (eps > 0.0) ? eps * eps * d0 : eps * eps;
    }
    __syncthreads();
    int r = 0;
    for (int k = 0; k < ell; ++k) {
        if (threadIdx.x == 0) {
            int jb = k;
            for (int j = k + 1; j < ell; ++j)
                if (A[piv[j] * ell + piv[j]] > A[piv[jb] * ell + piv[jb]]) jb = j;
            const int tmp = piv[k]; piv[k] = piv[jb]; piv[jb] = tmp;
            const double d = A[piv[k] * ell + piv[k]];
            s_stop = !(d > s_cut) ? 1 : (k >= cap ? 2 : 0);
            if (!s_stop) A[piv[k] * ell + piv[k]] = sqrt(d);
        }
        __syncthreads();
        if (s_stop) {
            if (s_stop == 2 && threadIdx.x == 0) atomicOr(flags + 1, 2);
            break;
        }
        const int pk = piv[k];
        const double rkk = A[pk * ell + pk];
        for (int j = k + 1 + threadIdx.x; j < ell; j += blockDim.x) A[pk * ell + piv[j]] /= rkk;
        __syncthreads();
        const int rem = ell - k - 1;
        for (int idx = threadIdx.x; idx < rem * rem; idx += blockDim.x) {
            const int i = k + 1 + idx % rem, j = k + 1 + idx / rem;
            if (i <= j) {
                const double v = A[piv[i] * ell + piv[j]] - A[pk * ell + piv[i]] * A[pk * ell + piv[j]];
                A[piv[i] * ell + piv[j]] = v;
                A[piv[j] * ell + piv[i]] = v;
            }
        }
        __syncthreads();
        r = k + 1;
    }
    // Xo[piv[j], c] = R[c][j] (j >= c);  Gm[piv[j], c] = (R11^-1)[j][c] (j <= c < r)
    for (int idx = threadIdx.x; idx < ell * r; idx += blockDim.x) {
        const int j = idx % ell, c = idx / ell;
        Xo[piv[j] + (int64_t)c * L] = (j >= c) ? A[piv[c] * ell + piv[j]] : 0.0;
        Gm[piv[j] + (int64_t)c * L] = 0.0;
    }
    __syncthreads();
    for (int c = threadIdx.x; c < r; c += blockDim.x) {   // column c of the upper-triangular inverse
        Gm[piv[c] + (int64_t)c * L] = 1.0 / A[piv[c] * ell + piv[c]];
        for (int i = c - 1; i >= 0; --i) {
            double acc = 0.0;
            for (int k2 = i + 1; k2 <= c; ++k2) acc += A[piv[i] * ell + piv[k2]] * Gm[piv[k2] + (int64_t)c * L];
            Gm[piv[i] + (int64_t)c * L] = -acc / A[piv[i] * ell + piv[i]];
        }
    }
    __syncthreads();
    return r;
}

// Randomized adaptive truncation, executed by nsub CTAs (sub = this CTA's index;
// sub 0 = leader).  The pieces are gathered once into contiguous stacks
// U_stack (m x K) and V_stack (q x K); every heavy pass is then a pipelined DMMA
// GEMM whose output tiles are spread over the group (gemm.cuh):
//   R2  T^T = Omega^T V_stack              (16 x K)
//   R3  Y   = U_stack T                    (m x 16)
//   R4  block classical Gram-Schmidt, twice (BCGS2): Y -= Q (Q^T Y) twice,
//       column-pivoted MGS of the block with the eps threshold (leader), the new
//       columns re-projected against the old basis and re-normalised
//   F1  P^T = Q^T U_stack                  (ell x K)
//   F2  W   = V_stack P                    (q x ell)   (= M^T Q)
//   F3  W = Q_W R (Householder), R^T = X' Z^T (one-sided Jacobi), rank (leader)
//   F4  U = Q X'(:, order),  V = W X'(:, order) Sigma^-2  (= Q_W Z)
// Work tiles are fixed, so the result does not depend on nsub.
static __device__ void trunc_rand(const TTask& t, int K, const TPiece* __restrict__ pieces, double* __restrict__ pool,
                                  int* __restrict__ ranks, int* __restrict__ flags, double eps,
                                  double* __restrict__ ctr, double* dsm, int sub, int nsub, int* bar,
                                  unsigned long long* stt) {
    // (nsub, bar: the group may shrink after the first round's probes, see below)
    const int m = t.m, q = t.q, cap = t.cap, np = t.piece_count;
    const int L = cap + TR_RB;
    const int Ks = t.kmax_tot;
    int rsplit = (nsub == t.nsub) ? trunc_rsplit(m, q, cap, Ks, t.nsub) : 1;
    bool rowsplit = nsub > 1 && (m + TR_RCH - 1) / TR_RCH >= nsub;   // R3 over owned rows
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int nchm = (m + TR_RCH - 1) / TR_RCH, nchq = (q + TR_RCH - 1) / TR_RCH;
    int om0, om1, oq0, oq1;                        // this CTA's own rows of the m- and q-sides
    own_rows(m, sub, nsub, om0, om1);
    own_rows(q, sub, nsub, oq0, oq1);
    TruncWs W = trunc_ws_layout(pool + t.ws, m, q, cap, Ks, t.nsub);
    int* ctl = (int*)W.ctl;                        // [0] done, [1] ell, [2] rank, [3] added, [8..] order
    double* gsm = dsm;                             // GEMM staging
    int* koff = (int*)((char*)dsm + TR_SMEM_A + ORDER_MAX * 4);   // TR_PMAX + 1 ints
    int* order = (int*)((char*)dsm + TR_SMEM_A);   // ORDER_MAX ints (leader, F3)
    __shared__ double scratch[32];
    __shared__ int s_added, s_rank, s_flag;
    __shared__ double s_ratio[TR_RB];
    __shared__ double s_scale[TR_PW];
    __shared__ double Gs[TR_RB * TR_RB], Rs[TR_RB * TR_RB];
    __shared__ int piv[TR_RB];
    __shared__ int s_na;
    __shared__ double s_maxn;
    int gen = 0;
    if (sub != 0) stt = nullptr;
    if (stt && threadIdx.x == 0) {
        unsigned long long now;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
        stt[0] = now;
    }
    if (np > TR_PMAX) {                            // planner guarantees np <= TR_PMAX
        if (threadIdx.x == 0 && sub == 0) atomicOr(flags + 1, 4);
        return;
    }
    if (threadIdx.x == 0) {
        int acc = 0;
        for (int p = 0; p < np; ++p) {
            koff[p] = acc;
            acc += dim_eval(pieces[t.piece_begin + p].w, ranks);
        }
        koff[np] = acc;
    }
    __syncthreads();
    // gather the stacks A = [alpha_p pad(U_p)] (m x K) and B = [pad(V_p)] (q x K): one warp per
    // (stacked column, 256-row block) item, 8 loads per lane, coalesced; GB items per warp in
    // flight (all loads, then all stores: one item at a time left the gather latency-bound)
    {
        constexpr int GB = 4;
        const int rbm = (m + 255) / 256, rbq = (q + 255) / 256;
        const int64_t nitem = (int64_t)K * (rbm + rbq);
        const int64_t wstride = (int64_t)nsub * nw;
        for (int64_t it0 = (int64_t)sub * nw + warp; it0 < nitem; it0 += GB * wstride) {
            double v[GB][8];
            double* dsts[GB];
            int r0s[GB], nrs[GB];
#pragma unroll
            for (int b2 = 0; b2 < GB; ++b2) {
                const int64_t it = it0 + b2 * wstride;
                dsts[b2] = nullptr;
                r0s[b2] = 0;
                nrs[b2] = 0;
#pragma unroll
                for (int u = 0; u < 8; ++u) v[b2][u] = 0.0;
                if (it < nitem) {
                    const int k = (int)(it / (rbm + rbq)), rb = (int)(it % (rbm + rbq));
                    const int p = piece_of(koff, np, k);
                    const TPiece& pc = pieces[t.piece_begin + p];
                    const int c = k - koff[p];
                    const bool isu = rb < rbm;
                    const int r0 = (isu ? rb : rb - rbm) * 256;
                    const int nr = isu ? m : q;
                    const int row0 = isu ? pc.u_row0 : pc.v_row0, rows = isu ? pc.u_rows : pc.v_rows;
                    const double al = isu ? pc.alpha : 1.0;
                    const double* src = pool + (isu ? pc.u_off + (int64_t)c * pc.u_ld : pc.v_off + (int64_t)c * pc.v_ld);
                    dsts[b2] = isu ? W.Ast + (int64_t)k * m : W.Bst + (int64_t)k * q;
                    r0s[b2] = r0;
                    nrs[b2] = nr;
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const int i = r0 + lane + 32 * u, ii = i - row0;
                        if (i < nr && ii >= 0 && ii < rows) v[b2][u] = al * __ldcg(src + ii);
                    }
                }
            }
#pragma unroll
            for (int b2 = 0; b2 < GB; ++b2) {
                if (dsts[b2] == nullptr) continue;
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int i = r0s[b2] + lane + 32 * u;
                    if (i < nrs[b2]) dsts[b2][i] = v[b2][u];
                }
            }
        }
    }
    double Srows = 0.0;                            // sum over stacked columns of (u_rows + v_rows)
    for (int p = 0; p < np; ++p)
        Srows += (double)(koff[p + 1] - koff[p]) * (pieces[t.piece_begin + p].u_rows + pieces[t.piece_begin + p].v_rows);
    const uint64_t seed = (uint64_t)t.u_out * 0x632BE59BD9B4E019ull;
    const GOp Ust = gop(W.Ast, m, false), Vst = gop(W.Bst, q, false);
    int ell = 0;
    double sest = 0.0;
    double flops = 0.0, bytes = 0.0;
    bool finished = false;
    for (int round = 0; !finished; ++round) {
        // ---- R1: TR_NB blocks of TR_RB Gaussian probes, Omega (q x TR_PW), in fixed row chunks
        for (int c = sub; c < nchq; c += nsub) {
            const int r0 = c * TR_RCH, r1 = min(q, r0 + TR_RCH);
            for (int idx = threadIdx.x; idx < (r1 - r0) * TR_PW; idx += blockDim.x) {
                const int i = r0 + idx % (r1 - r0), j = idx / (r1 - r0);
                W.Om[i + (int64_t)j * q] = rnd_normal(seed + (uint64_t)round * 0x100000000ull + (uint64_t)(i + j * q));
            }
        }
        coop_sync(bar, nsub, gen, stt);            // Omega (and the gathered stacks) complete
        {
            const int Kc = ((K + nsub - 1) / nsub + 15) & ~15;
            const int k0 = min(K, sub * Kc), k1 = min(K, k0 + Kc);
            // ---- R2: T^T = Omega^T V_stack  (TR_PW x K), one pass over the stack for all blocks
            // (few output tiles: inner dimension q split over the group, each CTA sums its own
            // R3 slice of T)
            if (rsplit > 1 && gemm_tiles(TR_PW, K, 64, 64) < nsub) {
                gemm_tn_rsplit(TR_PW, K, q, W.Om, q, W.Bst, q, W.Tt, TR_PW, W.Rpart, TR_PW, rsplit, sub, nsub, k0, k1,
                               bar, gen, stt, gsm);
                if (rowsplit) coop_sync(bar, nsub, gen, stt);   // the row-split R3 reads all of T
            } else {
                gemm_wide<true, false>(TR_PW, K, q, 1.0, gop(W.Om, q, true), Vst, 0.0, W.Tt, TR_PW, sub, nsub, gsm);
                coop_sync(bar, nsub, gen, stt);
            }
            // ---- R3: Y = U_stack T  (m x TR_PW), split over the stacked columns (each CTA one
            // 16-aligned slice, partials reduced on the owned 64-row chunks)
            // (tall blocks, at least one 64-row chunk per CTA: split over the owned row chunks
            // instead -- no partial sums)
            if (rowsplit) {
                if (om1 > om0)
                    gemm_wide<false, true>(om1 - om0, TR_PW, K, 1.0, gop(W.Ast + om0, m, false), gop(W.Tt, TR_PW, true), 0.0,
                                           W.Y + om0, m, 0, 1, gsm);
                __syncthreads();
            } else {
                double* Yp = (nsub == 1) ? W.Y : W.Ypart + (int64_t)sub * m * TR_PW;
                if (k1 > k0)
                    gemm_wide<false, true>(m, TR_PW, k1 - k0, 1.0, gop(W.Ast + (int64_t)k0 * m, m, false),
                              gop(W.Tt + (int64_t)k0 * TR_PW, TR_PW, true), 0.0, Yp, m, 0, 1, gsm);
                else
                    for (int idx = threadIdx.x; idx < m * TR_PW; idx += blockDim.x) Yp[idx] = 0.0;
                coop_sync(bar, nsub, gen, stt);
            }
        }
        flops += 4.0 * TR_PW * (double)K * (m + q);
        bytes += 8.0 * Srows;
        for (int c = om0 / TR_RCH; c * TR_RCH < om1; ++c) {
            const int r0 = c * TR_RCH, r1 = min(m, r0 + TR_RCH);
            if (nsub > 1 && !rowsplit) {
                for (int idx = threadIdx.x; idx < (r1 - r0) * TR_PW; idx += blockDim.x) {
                    const int64_t e = r0 + idx % (r1 - r0) + (int64_t)(idx / (r1 - r0)) * m;
                    double acc = 0.0;
                    for (int s2 = 0; s2 < nsub; ++s2) acc += __ldcg(W.Ypart + (int64_t)s2 * m * TR_PW + e);
                    W.Y[e] = acc;
                }
                __syncthreads();
            }
            for (int j = warp; j < TR_PW; j += nw) {
                double a = 0.0;
                for (int i = r0 + lane; i < r1; i += 32) a += W.Y[i + (int64_t)j * m] * W.Y[i + (int64_t)j * m];
                a = warp_sum(a);
                if (lane == 0) W.npart[(int64_t)c * TR_PW + j] = a;
            }
        }
        coop_sync(bar, nsub, gen, stt);
        // ---- shrink (first round): the row-owned middle (BCGS2) and the final products run
        // on nkeep CTAs (HM_TR_SHRINK 64-row chunks each); the others leave for other tasks
        // instead of waiting at the group's barriers.  A fresh barrier counter (bar + 1) takes over:
        // each kept CTA credits it with gen arrivals, so the generation count (and the stage
        // stamps) simply continue; partial buffers are indexed by sub < nkeep.
        if (TR_SHRINK > 0 && round == 0) {
            const int nkeep = min(nsub, (nchm + TR_SHRINK - 1) / TR_SHRINK);
            if (nkeep < nsub) {
                if (sub >= nkeep) return;
                nsub = nkeep;
                bar += 1;
                if (threadIdx.x == 0) atomicAdd(bar, gen);
                rsplit = 1;
                rowsplit = nsub > 1 && nchm >= nsub;
                own_rows(m, sub, nsub, om0, om1);
                own_rows(q, sub, nsub, oq0, oq1);
            }
        }
        // ---- scale: max_j ||M w_j|| over the probes seen so far (every CTA, same order)
        if (threadIdx.x < TR_PW) {
            const int j = threadIdx.x;
            double a = 0.0;
            for (int c = 0; c < nchm; ++c) a += __ldcg(W.npart + (int64_t)c * TR_PW + j);
            s_scale[j] = sqrt(a);
        }
        __syncthreads();
        for (int j = 0; j < TR_PW; ++j) sest = fmax(sest, s_scale[j]);
        const double thr = (eps > 0.0 ? eps * sest : -eps) * TR_STOP;
        __syncthreads();
        for (int blk = 0; blk < TR_NB && !finished; ++blk) {
            double* Yb = W.Y + (int64_t)blk * TR_RB * m;
        // ---- R4 (row-owned, no leader loops): BCGS2 with a pivoted Cholesky-QR of the block
        //   Y <- (I - Q Q^T) Y twice; G = Y^T Y; pivoted Cholesky of G with the
        //   threshold -> selection P, R; Qn = Y_P R^-1; Qn <- (I - Q Q^T) Qn; CholQR of Qn.
        // Partial reductions over each CTA's own 64-row chunks are summed by every CTA
        // in the same order, so all CTAs take the same decisions without a broadcast.
        if (ell > 0) {
            for (int pass = 0; pass < 2; ++pass) proj_owned(W, m, ell, L, Yb, TR_RB, sub, nsub, om0, om1, bar, gen, stt, gsm);
            flops += 8.0 * TR_RB * (double)ell * m;
        }
        gram_owned(W, m, Yb, TR_RB, sub, nsub, om0, om1, bar, gen, stt, gsm, Gs);
        // pivoted Cholesky (redundant, identical in every CTA): accept pivots above
        // max(thr, 1e-4 * largest) so R stays well conditioned (cond <= 1e4); weaker
        // directions are picked up by the next round's probes
        // (warp 0: lanes own pivot candidates / Schur entries; same arithmetic, per entry, as a
        // serial loop, ties of the pivot search to the lowest index)
        if (warp == 0) {
            double dg = (lane < TR_RB) ? Gs[lane * TR_RB + lane] : 0.0;
            if (lane < TR_RB) piv[lane] = lane;
            double d0 = dg;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) d0 = fmax(d0, __shfl_xor_sync(0xffffffffu, d0, o));
            const double cut = fmax(thr * thr, 1e-8 * d0);
            if (lane == 0) s_maxn = sqrt(fmax(d0, 0.0));
            __syncwarp();
            int na = 0;
            for (int k = 0; k < TR_RB && ell + k < L; ++k) {
                // argmax over j >= k of the remaining diagonal (lowest j on ties)
                double bv = (lane >= k && lane < TR_RB) ? Gs[piv[lane] * TR_RB + piv[lane]] : -DBL_MAX;
                int bj = (lane >= k && lane < TR_RB) ? lane : TR_RB;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
                    const int oj = __shfl_xor_sync(0xffffffffu, bj, o);
                    if (ov > bv || (ov == bv && oj < bj)) { bv = ov; bj = oj; }
                }
                __syncwarp();
                if (lane == 0) { const int tmp = piv[k]; piv[k] = piv[bj]; piv[bj] = tmp; }
                __syncwarp();
                const int pk = piv[k];
                const double d = Gs[pk * TR_RB + pk];
                if (!(d > cut)) break;
                const double rkk = sqrt(d);
                if (lane == k) Rs[k * TR_RB + k] = rkk;
                if (lane > k && lane < TR_RB) Rs[k * TR_RB + lane] = Gs[pk * TR_RB + piv[lane]] / rkk;
                __syncwarp();
                const int rem = TR_RB - k - 1;   // trailing Schur complement (pivoted indices), both triangles
                for (int idx = lane; idx < rem * rem; idx += 32) {
                    const int i = k + 1 + idx % rem, j = k + 1 + idx / rem;
                    Gs[piv[i] * TR_RB + piv[j]] -= Rs[k * TR_RB + i] * Rs[k * TR_RB + j];
                }
                __syncwarp();
                ++na;
            }
            if (lane == 0) s_na = na;
        }
        __syncthreads();
        const int na = s_na;
        const double maxn = s_maxn;
        if (na > 0) {
            // Qn = Y_P R^-1 on the owned rows (thread per row, forward substitution)
            {
                const int r0 = om0, r1 = om1;
                for (int i = r0 + threadIdx.x; i < r1; i += blockDim.x) {
                    double x[TR_RB];
#pragma unroll
                    for (int j = 0; j < TR_RB; ++j) {
                        if (j < na) {
                            double v = Yb[i + (int64_t)piv[j] * m];
                            for (int k = 0; k < j; ++k) v -= x[k] * Rs[k * TR_RB + j];
                            x[j] = v / Rs[j * TR_RB + j];
                            W.Q[i + (int64_t)(ell + j) * m] = x[j];
                        }
                    }
                }
            }
            __syncthreads();
            double* Qn = W.Q + (int64_t)ell * m;
            if (ell > 0) proj_owned(W, m, ell, L, Qn, na, sub, nsub, om0, om1, bar, gen, stt, gsm);
            gram_owned(W, m, Qn, na, sub, nsub, om0, om1, bar, gen, stt, gsm, Gs);
            // CholQR of the (nearly orthonormal) new block: Qn <- Qn chol(Qn^T Qn)^-1
            // (warp 0: lane j forms row k's entry j; sums in the order l = 0 .. k-1)
            if (warp == 0) {
                for (int k = 0; k < na; ++k) {
                    double v = 0.0;
                    if (lane >= k && lane < na) {
                        v = Gs[k * TR_RB + lane];
                        for (int l = 0; l < k; ++l) v -= Rs[l * TR_RB + k] * Rs[l * TR_RB + lane];
                    }
                    const double rkk = sqrt(fmax(__shfl_sync(0xffffffffu, v, k), 1e-300));
                    if (lane == k) Rs[k * TR_RB + k] = rkk;
                    if (lane > k && lane < na) Rs[k * TR_RB + lane] = v / rkk;
                    __syncwarp();
                }
            }
            __syncthreads();
            {
                const int r0 = om0, r1 = om1;
                for (int i = r0 + threadIdx.x; i < r1; i += blockDim.x) {
                    double x[TR_RB];
#pragma unroll
                    for (int j = 0; j < TR_RB; ++j) {
                        if (j < na) {
                            double v = Qn[i + (int64_t)j * m];
                            for (int k = 0; k < j; ++k) v -= x[k] * Rs[k * TR_RB + j];
                            x[j] = v / Rs[j * TR_RB + j];
                            Qn[i + (int64_t)j * m] = x[j];
                        }
                    }
                }
            }
            __syncthreads();
            flops += 4.0 * (double)na * ell * m + 6.0 * (double)na * na * m;
        }
        const int ell2 = ell + na;
        bool done = (maxn <= thr) || na == 0;
        if (!done && ell2 >= L) { done = true; if (sub == 0 && threadIdx.x == 0) atomicOr(flags + 1, 2); }
        if (!done && (ell2 >= m || ell2 >= q)) done = true;
        ell = ell2;
        if (done || round > 64) finished = true;
        __syncthreads();
        }
    }
    if (stt && threadIdx.x == 0) { stt[62] = (unsigned long long)K; stt[63] = (unsigned long long)ell; }
    coop_sync(bar, nsub, gen, stt);                // basis Q complete on every row
    if (ell == 0) {
        if (sub == 0 && threadIdx.x == 0) {
            ranks[t.rslot] = 0;
            atomicAdd(ctr + CTR_TRUNC + 0, flops);
            atomicAdd(ctr + CTR_TRUNC + 1, bytes);
        }
        coop_sync(bar, nsub, gen, stt);
        return;
    }
    // ---- F1: P^T = Q^T U_stack  (ell x K);  F2: W = V_stack P  (q x ell)
    if (rsplit > 1 && gemm_tiles(ell, K, 64, 64) < nsub) {
        const int Kc = ((K + nsub - 1) / nsub + 15) & ~15;
        const int k0 = min(K, sub * Kc), k1 = min(K, k0 + Kc);
        gemm_tn_rsplit(ell, K, m, W.Q, m, W.Ast, m, W.Pt, L, W.Rpart, L, rsplit, sub, nsub, k0, k1, bar, gen, stt,
                       gsm);
        if (!(nsub > 1 && q <= TR_WSPLIT_Q)) coop_sync(bar, nsub, gen, stt);   // F2 below reads all of P
    } else {
        gemm_wide<true, false>(ell, K, m, 1.0, gop(W.Q, m, true), Ust, 0.0, W.Pt, L, sub, nsub, gsm);
        coop_sync(bar, nsub, gen, stt);
    }
    if (nsub > 1 && q <= TR_WSPLIT_Q) {            // split over the stacked columns, reduce owned rows
        const int Kc = ((K + nsub - 1) / nsub + 15) & ~15;
        const int k0 = min(K, sub * Kc), k1 = min(K, k0 + Kc);
        double* Wp = W.Wpart + (int64_t)sub * q * L;
        if (k1 > k0)
            gemm_wide<false, true>(q, ell, k1 - k0, 1.0, gop(W.Bst + (int64_t)k0 * q, q, false), gop(W.Pt + (int64_t)k0 * L, L, true),
                      0.0, Wp, q, 0, 1, gsm);
        else
            for (int idx = threadIdx.x; idx < q * ell; idx += blockDim.x) Wp[idx] = 0.0;
        coop_sync(bar, nsub, gen, stt);
        for (int c = sub; c < nchq; c += nsub) {
            const int r0 = c * TR_RCH, r1 = min(q, r0 + TR_RCH);
            for (int idx = threadIdx.x; idx < (r1 - r0) * ell; idx += blockDim.x) {
                const int64_t e = r0 + idx % (r1 - r0) + (int64_t)(idx / (r1 - r0)) * q;
                double acc = 0.0;
                for (int s2 = 0; s2 < nsub; ++s2) acc += __ldcg(W.Wpart + (int64_t)s2 * q * L + e);
                W.Wm[e] = acc;
            }
        }
    } else {
        gemm_wide<false, true>(q, ell, K, 1.0, Vst, gop(W.Pt, L, true), 0.0, W.Wm, q, sub, nsub, gsm);
    }
    coop_sync(bar, nsub, gen, stt);
    flops += 4.0 * (double)ell * K * (m + q);
    bytes += 8.0 * Srows;
    const int Kw = min(q, ell);
    const bool gram = fabs(eps) >= TR_GRAM_EPS;
    if (gram) {
        // ---- F3 (Gram path, eps >= TR_GRAM_EPS): G = W^T W (partials spread over the group),
        // then a column-pivoted Cholesky of G stopped at eps^2 * max diag (gram_pchol): a
        // rank-revealing factorisation, resolving sigma_i / sigma_1 down to ~1e-8 -- enough
        // for eps >= 1e-7 -- at a fraction of the cost of an iterative eigensolver.
        double* Gp = W.Gp2 + (int64_t)sub * L * L;
        if (oq1 > oq0)
            gemm_wide<true, false>(ell, ell, oq1 - oq0, 1.0, gop(W.Wm + oq0, q, true), gop(W.Wm + oq0, q, false), 0.0, Gp,
                                   L, 0, 1, gsm);
        else
            for (int idx = threadIdx.x; idx < ell * ell; idx += blockDim.x) Gp[(idx % ell) + (int64_t)(idx / ell) * L] = 0.0;
        coop_sync(bar, nsub, gen, stt);
        for (int idx = sub * blockDim.x + threadIdx.x; idx < ell * ell; idx += nsub * blockDim.x) {
            const int64_t e = (idx % ell) + (int64_t)(idx / ell) * L;
            double acc = 0.0;
            for (int s2 = 0; s2 < nsub; ++s2) acc += __ldcg(W.Gp2 + (int64_t)s2 * L * L + e);
            W.S[idx] = acc;                        // ell x ell, ld ell
        }
        coop_sync(bar, nsub, gen, stt);
        flops += 2.0 * (double)ell * ell * q;
    }
    if (sub == 0 && gram) {
        const int r = gram_pchol(W.S, ell, eps, cap, W.Xo, W.G, L, gsm, order, flags);
        if (threadIdx.x == 0) ctl[2] = r;
        flops += (double)ell * ell * ell / 3.0;
    }
    if (sub == 0 && !gram) {
        {
            // ---- F3 (Householder path): QR of a copy of W, S = R^T, Jacobi S Z = X'
            for (int idx = threadIdx.x; idx < q * ell; idx += blockDim.x) W.Wc[idx] = W.Wm[idx];
            __syncthreads();
            house_qr(W.Wc, q, ell, W.tau, W.sig);   // (sig: scratch here, filled below)
            for (int idx = threadIdx.x; idx < ell * Kw; idx += blockDim.x) {
                const int i = idx % ell, j = idx / ell;
                W.S[i + (int64_t)j * ell] = (i >= j) ? W.Wc[j + (int64_t)i * q] : 0.0;
            }
            __syncthreads();
            jacobi_smem(W.S, ell, Kw, W.Z, gsm, &s_flag);
        }
        const int kdim = Kw;
        for (int j = warp; j < kdim; j += nw) {
            double sacc = 0.0;
            for (int r = lane; r < ell; r += 32) sacc += W.S[r + (int64_t)j * ell] * W.S[r + (int64_t)j * ell];
            sacc = warp_sum(sacc);
            if (lane == 0) W.sig[j] = sqrt(sacc);
        }
        __syncthreads();
        const int kk = min(kdim, ORDER_MAX);
        for (int j = threadIdx.x; j < kk; j += blockDim.x) {
            int pos = 0;
            const double sj = W.sig[j];
            for (int b2 = 0; b2 < kk; ++b2) pos += (W.sig[b2] > sj || (W.sig[b2] == sj && b2 < j)) ? 1 : 0;
            order[pos] = j;
        }
        __syncthreads();
        {
            const double smax = W.sig[order[0]];
            int cnt = 0;
            for (int j = threadIdx.x; j < kk; j += blockDim.x) cnt += (W.sig[j] > tr_cut(eps, smax) && W.sig[j] > 0.0) ? 1 : 0;
            const double tot = block_sum((double)cnt, scratch);
            if (threadIdx.x == 0) {
                int r = (int)(tot + 0.5);
                if (r > cap) { atomicOr(flags + 1, 2); r = cap; }
                s_rank = r;
                ctl[2] = r;
            }
        }
        __syncthreads();
        const int r = s_rank;
        for (int idx = threadIdx.x; idx < ell * r; idx += blockDim.x) {
            const int l = idx % ell, c = idx / ell;
            const int oc = order[c];
            // Xo = X'(:, order), G = Xo / sigma^2
            const double x = W.S[l + (int64_t)oc * ell];
            const double sg = W.sig[oc];
            W.Xo[l + (int64_t)c * L] = x;
            W.G[l + (int64_t)c * L] = x / (sg * sg);
        }
        const double el = ell, qd = q, kw = Kw;
        flops += 2.0 * (qd * el * kw - kw * kw * kw / 3.0) + 3.0 * kw * (kw - 1.0) * (el + kw);
    }
    coop_sync(bar, nsub, gen, stt);                // rank, Xo, G published
    const int r = __ldcg(ctl + 2);
    // ---- F4: U_out = Q Xo (m x r),  V_out = W G (q x r)
    double* Uo = pool + t.u_out;
    double* Vo = pool + t.v_out;
    if (r > 0) {
        // tiles of the V product start where the U tiles left off, so idle CTAs take them first
        const int tu = gemm_tiles(m, r, 64, 64);
        gemm_wide<false, false>(m, r, ell, 1.0, gop(W.Q, m, false), gop(W.Xo, L, false), 0.0, Uo, m, sub, nsub, gsm);
        gemm_wide<false, false>(q, r, ell, 1.0, gop(W.Wm, q, false), gop(W.G, L, false), 0.0, Vo, q, (sub + tu) % nsub, nsub, gsm);
    }
    if (sub == 0 && threadIdx.x == 0) {
        flops += 2.0 * (double)r * ell * (m + q);
        bytes += 8.0 * (double)r * (m + q);
        atomicAdd(ctr + CTR_TRUNC + 0, flops);
        atomicAdd(ctr + CTR_TRUNC + 1, bytes);
    }
    coop_sync(bar, nsub, gen, stt);                // all output rows written before the leader publishes
    if (sub == 0 && threadIdx.x == 0) ranks[t.rslot] = r;
}

// dynamic shared memory (bytes) the truncation needs
constexpr int TR_SMEM_R = TR_SMEM_A + ORDER_MAX * 4 + (TR_PMAX + 1) * 4;
constexpr int TR_SMEM_X = TR_XS_OFF * 8 + TR_XS_DOUBLES * 8;
constexpr int TR_SMEM = TR_SMEM_R > TR_SMEM_X ? TR_SMEM_R : TR_SMEM_X;

// sub / nsub / bar: this CTA's index in a cooperative truncation (nsub CTAs,
// persistent executor only), else 0 / 1 / nullptr
__device__ __forceinline__ void trunc_run(const TTask& t, const TPiece* __restrict__ pieces, double* pool, int* ranks,
                                          int* flags, double eps, double* ctr, double* dsm, int sub = 0, int nsub = 1,
                                          int* bar = nullptr, unsigned long long* stt = nullptr) {
    int K = 0;
    for (int p = 0; p < t.piece_count; ++p) K += dim_eval(pieces[t.piece_begin + p].w, ranks);
    eps *= t.eps_scale;   // keeps the sign: > 0 relative, < 0 absolute
    if (trunc_exact_path(t.m, t.q, t.kmax_tot)) trunc_exact(t, K, pieces, pool, ranks, flags, eps, ctr, dsm);
    else trunc_rand(t, K, pieces, pool, ranks, flags, eps, ctr, dsm, sub, nsub, bar, stt);
}

}  // namespace hm
