// Low-rank truncation kernel k_trunc ("efficient rank-truncation
// techniques"; adaptive-rank strategy of Remark 2, l.166, reading R4):
//
//   B <- best rank-r approximation, sigma_i > eps * sigma_1, of
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
//    twice-projected against the basis Q, stop when every projected probe has
//    norm <= eps * sigma_est / 8 (so ||M - Q Q^T M|| <= eps sigma_1 with
//    probability >= 1 - 10^-RB); then W = M^T Q (again piece by piece),
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

namespace hm {

constexpr int TR_THREADS = 256;
constexpr int ORDER_MAX = 512;

// Householder QR of A (m x K, ld m) in place; tau[K].  R in the upper triangle.
static __device__ __noinline__ void house_qr(double* A, int m, int K, double* tau, double* scratch) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int kmin = min(m, K);
    __shared__ double s_beta, s_scale, s_tau;
    for (int i = 0; i < kmin; ++i) {
        double* a = A + (int64_t)i * m;
        double ss = 0.0;
        for (int r = i + 1 + threadIdx.x; r < m; r += blockDim.x) ss += a[r] * a[r];
        const double sig = block_sum(ss, scratch);
        if (threadIdx.x == 0) {
            const double alpha = a[i];
            if (sig == 0.0) {
                s_tau = 0.0;
                s_scale = 0.0;
                s_beta = alpha;
            } else {
                const double nrm = sqrt(alpha * alpha + sig);
                const double beta = (alpha <= 0.0) ? nrm : -nrm;
                s_tau = (beta - alpha) / beta;
                s_scale = 1.0 / (alpha - beta);
                s_beta = beta;
            }
            tau[i] = s_tau;
        }
        __syncthreads();
        const double tv = s_tau, sc = s_scale;
        if (tv != 0.0)
            for (int r = i + 1 + threadIdx.x; r < m; r += blockDim.x) a[r] *= sc;
        __syncthreads();
        if (threadIdx.x == 0) a[i] = s_beta;
        __syncthreads();
        if (tv != 0.0) {
            // apply H = I - tau v v^T (v_i = 1) to columns c > i: one warp per column
            for (int c = i + 1 + warp; c < K; c += nw) {
                double* col = A + (int64_t)c * m;
                double w = (lane == 0) ? col[i] : 0.0;
                for (int r = i + 1 + lane; r < m; r += 32) w += a[r] * col[r];
                w = warp_sum(w) * tv;
                if (lane == 0) col[i] -= w;
                for (int r = i + 1 + lane; r < m; r += 32) col[r] -= w * a[r];
            }
        }
        __syncthreads();
    }
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

// one-sided Jacobi: X (rows x n, ld rows) -> X Z with orthogonal columns; Z (n x n, ld n)
static __device__ __noinline__ void jacobi_svd(double* X, int rows, int n, double* Z, int* s_flag) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int idx = threadIdx.x; idx < n * n; idx += blockDim.x) Z[idx] = ((idx % n) == (idx / n)) ? 1.0 : 0.0;
    __syncthreads();
    if (n < 2) return;
    const int nn = (n + 1) & ~1;   // even number of players (one dummy if n odd)
    for (int sweep = 0; sweep < 40; ++sweep) {
        if (threadIdx.x == 0) *s_flag = 0;
        __syncthreads();
        for (int round = 0; round < nn - 1; ++round) {
            for (int pr = warp; pr < nn / 2; pr += nw) {
                // round-robin pairing: player 0 fixed, others rotate
                int a = (pr == 0) ? 0 : ((round + pr - 1) % (nn - 1)) + 1;
                int b = ((round + nn - 2 - pr) % (nn - 1)) + 1;
                if (pr == 0) b = ((round + nn - 2) % (nn - 1)) + 1;
                if (a >= n || b >= n) continue;
                if (a > b) { int tmp = a; a = b; b = tmp; }
                double* xa = X + (int64_t)a * rows;
                double* xb = X + (int64_t)b * rows;
                double al = 0.0, be = 0.0, ga = 0.0;
                for (int r = lane; r < rows; r += 32) {
                    const double u = xa[r], v = xb[r];
                    al += u * u; be += v * v; ga += u * v;
                }
                al = warp_sum(al); be = warp_sum(be); ga = warp_sum(ga);
                if (fabs(ga) > 1e-15 * sqrt(al * be) && ga != 0.0) {
                    const double zeta = (be - al) / (2.0 * ga);
                    const double tt = ((zeta >= 0.0) ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                    const double c = 1.0 / sqrt(1.0 + tt * tt), s = c * tt;
                    for (int r = lane; r < rows; r += 32) {
                        const double u = xa[r], v = xb[r];
                        xa[r] = c * u - s * v;
                        xb[r] = s * u + c * v;
                    }
                    double* za = Z + (int64_t)a * n;
                    double* zb = Z + (int64_t)b * n;
                    for (int r = lane; r < n; r += 32) {
                        const double u = za[r], v = zb[r];
                        za[r] = c * u - s * v;
                        zb[r] = s * u + c * v;
                    }
                    if (lane == 0) *s_flag = 1;
                }
            }
            __syncthreads();
        }
        if (*s_flag == 0) break;
        __syncthreads();
    }
    __syncthreads();
}


// ---------------------------------------------------------------- exact path
static __device__ void trunc_exact(const TTask& t, int K, const TPiece* __restrict__ pieces, double* __restrict__ pool,
                            int* __restrict__ ranks, int* __restrict__ flags, double eps, double* __restrict__ ctr,
                            double* dsm) {
    __shared__ double scratch[32];
    int* order = (int*)dsm;                        // ORDER_MAX ints (dynamic shared memory)
    __shared__ int s_flag;
    __shared__ int s_rank;
    const int m = t.m, q = t.q;
    double* ws = pool + t.ws;
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
        for (int idx = threadIdx.x; idx < m * w; idx += blockDim.x) {
            const int r = idx % m, c = idx / m;
            const int rr = r - pc.u_row0;
            A[(int64_t)(koff + c) * m + r] = (rr >= 0 && rr < pc.u_rows) ? pc.alpha * Up[rr + (int64_t)c * pc.u_ld] : 0.0;
        }
        for (int idx = threadIdx.x; idx < q * w; idx += blockDim.x) {
            const int r = idx % q, c = idx / q;
            const int rr = r - pc.v_row0;
            Bm[(int64_t)(koff + c) * q + r] = (rr >= 0 && rr < pc.v_rows) ? Vp[rr + (int64_t)c * pc.v_ld] : 0.0;
        }
        koff += w;
    }
    __syncthreads();
    if (K == 0) {
        if (threadIdx.x == 0) ranks[t.rslot] = 0;
        return;
    }
    house_qr(A, m, K, tauA, scratch);
    house_qr(Bm, q, K, tauB, scratch);
    const int Ka = min(m, K), Kb = min(q, K);
    // X = R_A R_B^T  (Ka x Kb), R_A[i][c] (c >= i) = A[i + c m], R_B[j][c] = Bm[j + c q]
    for (int idx = threadIdx.x; idx < Ka * Kb; idx += blockDim.x) {
        const int i = idx % Ka, j = idx / Ka;
        double s = 0.0;
        for (int c = max(i, j); c < K; ++c) s += A[i + (int64_t)c * m] * Bm[j + (int64_t)c * q];
        X[i + (int64_t)j * Ka] = s;
    }
    __syncthreads();
    jacobi_svd(X, Ka, Kb, Z, &s_flag);
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
        for (int j = threadIdx.x; j < kk; j += blockDim.x) cnt += (sig[j] > eps * s_smax && sig[j] > 0.0) ? 1 : 0;
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

static __device__ void trunc_rand(const TTask& t, int K, const TPiece* __restrict__ pieces, double* __restrict__ pool,
                           int* __restrict__ ranks, int* __restrict__ flags, double eps, double* __restrict__ ctr,
                           double* dsm) {
    const int m = t.m, q = t.q, cap = t.cap;
    const int L = cap + TR_RB;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    double* ws = pool + t.ws;
    double* Om = ws;                              // q x RB
    double* Qm = Om + (int64_t)q * TR_RB;          // m x L
    double* Yn = Qm + (int64_t)m * L;              // m x RB
    double* Wm = Yn + (int64_t)m * TR_RB;          // q x L
    double* Pp = Wm + (int64_t)q * L;              // wmax x L
    double* S = Pp + (int64_t)t.wmax * L;          // L x L
    double* Z = S + (int64_t)L * L;                // L x L
    double* tau = Z + (int64_t)L * L;              // L
    double* sig = tau + L;                         // L
    double* Tp = dsm;                              // per-piece T_p = V_p^T Omega (TR_WMAX_SM x RB)
    double* Cs = Tp + TR_WMAX_SM * TR_RB;          // Q^T Y  (TR_LMAX x RB)
    __shared__ double scratch[32];
    __shared__ int s_added, s_rank, s_flag;
    __shared__ double s_ratio[TR_RB];
    __shared__ int s_alive[TR_RB];
    int* order = (int*)(Cs + TR_LMAX * TR_RB);     // ORDER_MAX ints
    const uint64_t seed = (uint64_t)t.u_out * 0x632BE59BD9B4E019ull;
    int ell = 0;
    double sest = 0.0;
    double flops = 0.0, bytes = 0.0;
    for (int round = 0;; ++round) {
        // ---- probes Omega (q x RB) and zero Yn
        for (int idx = threadIdx.x; idx < q * TR_RB; idx += blockDim.x)
            Om[idx] = rnd_normal(seed + (uint64_t)round * 0x100000000ull + (uint64_t)idx);
        for (int idx = threadIdx.x; idx < m * TR_RB; idx += blockDim.x) Yn[idx] = 0.0;
        __syncthreads();
        // ---- Yn = M Omega = sum_p alpha_p U_p (V_p^T Omega_rows)
        for (int pi = 0; pi < t.piece_count; ++pi) {
            const TPiece pc = pieces[t.piece_begin + pi];
            const int w = dim_eval(pc.w, ranks);
            if (w == 0) continue;
            const double* U = pool + pc.u_off;
            const double* V = pool + pc.v_off;
            for (int c0 = 0; c0 < w; c0 += TR_WMAX_SM) {
                const int wc = min(TR_WMAX_SM, w - c0);
                for (int c = warp; c < wc; c += nw) {
                    double acc[TR_RB];
#pragma unroll
                    for (int j = 0; j < TR_RB; ++j) acc[j] = 0.0;
                    const double* vc = V + (int64_t)(c0 + c) * pc.v_ld;
                    for (int i = lane; i < pc.v_rows; i += 32) {
                        const double v = vc[i];
                        const double* o = Om + pc.v_row0 + i;
#pragma unroll
                        for (int j = 0; j < TR_RB; ++j) acc[j] += v * o[(int64_t)j * q];
                    }
                    warp_sum_arr(acc);
                    if (lane == 0)
#pragma unroll
                        for (int j = 0; j < TR_RB; ++j) Tp[c + j * TR_WMAX_SM] = acc[j];
                }
                __syncthreads();
                for (int i = threadIdx.x; i < pc.u_rows; i += blockDim.x) {
                    double acc[TR_RB];
#pragma unroll
                    for (int j = 0; j < TR_RB; ++j) acc[j] = 0.0;
                    for (int c = 0; c < wc; ++c) {
                        const double u = U[i + (int64_t)(c0 + c) * pc.u_ld];
#pragma unroll
                        for (int j = 0; j < TR_RB; ++j) acc[j] += u * Tp[c + j * TR_WMAX_SM];
                    }
                    double* y = Yn + pc.u_row0 + i;
#pragma unroll
                    for (int j = 0; j < TR_RB; ++j) y[(int64_t)j * m] += pc.alpha * acc[j];
                }
                __syncthreads();
            }
            flops += 4.0 * TR_RB * w * (double)(pc.u_rows + pc.v_rows);
            bytes += 8.0 * w * (double)(pc.u_rows + pc.v_rows);
        }
        // ---- sigma_1 lower bound: max_j ||Y_j|| / ||Omega_j||  (one warp per probe)
        for (int j = warp; j < TR_RB; j += nw) {
            double a = 0.0, b = 0.0;
            for (int i = lane; i < m; i += 32) a += Yn[i + (int64_t)j * m] * Yn[i + (int64_t)j * m];
            for (int i = lane; i < q; i += 32) b += Om[i + (int64_t)j * q] * Om[i + (int64_t)j * q];
            a = warp_sum(a);
            b = warp_sum(b);
            if (lane == 0) s_ratio[j] = (b > 0.0) ? sqrt(a / b) : 0.0;
        }
        __syncthreads();
        for (int j = 0; j < TR_RB; ++j) sest = fmax(sest, s_ratio[j]);
        const double thr = eps * sest * 0.125;
        // ---- Yn <- (I - Q Q^T) Yn, twice
        if (ell > 0) {
            for (int pass = 0; pass < 2; ++pass) {
                for (int l = warp; l < ell; l += nw) {
                    double acc[TR_RB];
#pragma unroll
                    for (int j = 0; j < TR_RB; ++j) acc[j] = 0.0;
                    const double* ql = Qm + (int64_t)l * m;
                    for (int i = lane; i < m; i += 32) {
                        const double qv = ql[i];
#pragma unroll
                        for (int j = 0; j < TR_RB; ++j) acc[j] += qv * Yn[i + (int64_t)j * m];
                    }
                    warp_sum_arr(acc);
                    if (lane == 0)
#pragma unroll
                        for (int j = 0; j < TR_RB; ++j) Cs[l + j * TR_LMAX] = acc[j];
                }
                __syncthreads();
                for (int i = threadIdx.x; i < m; i += blockDim.x) {
                    double acc[TR_RB];
#pragma unroll
                    for (int j = 0; j < TR_RB; ++j) acc[j] = 0.0;
                    for (int l = 0; l < ell; ++l) {
                        const double qv = Qm[i + (int64_t)l * m];
#pragma unroll
                        for (int j = 0; j < TR_RB; ++j) acc[j] += qv * Cs[l + j * TR_LMAX];
                    }
#pragma unroll
                    for (int j = 0; j < TR_RB; ++j) Yn[i + (int64_t)j * m] -= acc[j];
                }
                __syncthreads();
            }
            flops += 8.0 * TR_RB * (double)ell * m;
        }
        // ---- column-pivoted MGS of the RB probes with re-orthogonalisation: take the
        // probe with the largest residual norm while it exceeds thr, normalise it,
        // project it out of the remaining probes (twice).  When it stops, every
        // remaining probe residual is <= thr -- the certificate of the range finder.
        if (threadIdx.x == 0) s_added = 0;
        for (int j = threadIdx.x; j < TR_RB; j += blockDim.x) s_alive[j] = 1;
        __syncthreads();
        double maxn = 0.0;
        for (int step = 0; step < TR_RB; ++step) {
            for (int j = warp; j < TR_RB; j += nw) {
                double a = 0.0;
                if (s_alive[j])
                    for (int i = lane; i < m; i += 32) a += Yn[i + (int64_t)j * m] * Yn[i + (int64_t)j * m];
                a = warp_sum(a);
                if (lane == 0) s_ratio[j] = s_alive[j] ? sqrt(a) : -1.0;
            }
            __syncthreads();
            int jp = -1;
            double best = -1.0;
            for (int j = 0; j < TR_RB; ++j)
                if (s_ratio[j] > best) { best = s_ratio[j]; jp = j; }
            if (step == 0) maxn = best;
            const int na = s_added;
            if (!(best > thr) || ell + na >= L) break;
            // re-orthogonalise the pivot against the whole basis (old + new), twice:
            // its residual can be ~eps below its original norm, so the rounding of
            // the earlier projections must be removed before normalising
            double* yp = Yn + (int64_t)jp * m;
            const int nb = ell + na;
            for (int pass = 0; pass < 2 && nb > 0; ++pass) {
                for (int l = warp; l < nb; l += nw) {
                    const double* ql = Qm + (int64_t)l * m;
                    double d = 0.0;
                    for (int i = lane; i < m; i += 32) d += ql[i] * yp[i];
                    d = warp_sum(d);
                    if (lane == 0) Cs[l] = d;
                }
                __syncthreads();
                for (int i = threadIdx.x; i < m; i += blockDim.x) {
                    double a = 0.0;
                    for (int l = 0; l < nb; ++l) a += Qm[i + (int64_t)l * m] * Cs[l];
                    yp[i] -= a;
                }
                __syncthreads();
            }
            double nn = 0.0;
            for (int i = threadIdx.x; i < m; i += blockDim.x) nn += yp[i] * yp[i];
            const double nrm = sqrt(block_sum(nn, scratch));
            if (!(nrm > thr)) {                    // only rounding left: drop the probe
                if (threadIdx.x == 0) s_alive[jp] = 0;
                __syncthreads();
                continue;
            }
            double* qn = Qm + (int64_t)(ell + na) * m;
            const double inv = 1.0 / nrm;
            for (int i = threadIdx.x; i < m; i += blockDim.x) qn[i] = yp[i] * inv;
            __syncthreads();
            if (threadIdx.x == 0) { s_alive[jp] = 0; s_added = na + 1; }
            for (int j = warp; j < TR_RB; j += nw) {
                if (j == jp || !s_alive[j]) continue;
                double* y = Yn + (int64_t)j * m;
                for (int pass = 0; pass < 2; ++pass) {
                    double d = 0.0;
                    for (int i = lane; i < m; i += 32) d += qn[i] * y[i];
                    d = warp_sum(d);
                    for (int i = lane; i < m; i += 32) y[i] -= d * qn[i];
                    __syncwarp();
                }
            }
            __syncthreads();
        }
        const int added = s_added;
        flops += 4.0 * m * (double)TR_RB * TR_RB;
        ell += added;
        if (maxn <= thr || added == 0) break;      // every probe below eps sigma_est / 8
        if (ell >= L) {                            // basis full: no room to certify the tolerance
            if (threadIdx.x == 0) atomicOr(flags + 1, 2);
            break;
        }
        if (ell >= m || ell >= q) break;           // basis spans the whole range
    }
    __syncthreads();
    if (ell == 0) {
        if (threadIdx.x == 0) {
            ranks[t.rslot] = 0;
            atomicAdd(ctr + CTR_TRUNC + 0, flops);
            atomicAdd(ctr + CTR_TRUNC + 1, bytes);
        }
        return;
    }
    // ---- W = M^T Q = sum_p alpha_p V_p (U_p^T Q_rows)   (q x ell)
    for (int idx = threadIdx.x; idx < q * ell; idx += blockDim.x) Wm[idx] = 0.0;
    __syncthreads();
    for (int pi = 0; pi < t.piece_count; ++pi) {
        const TPiece pc = pieces[t.piece_begin + pi];
        const int w = dim_eval(pc.w, ranks);
        if (w == 0) continue;
        const double* U = pool + pc.u_off;
        const double* V = pool + pc.v_off;
        // P_p[c, l] = alpha * sum_i U[i, c] Q[u_row0 + i, l]   (w x ell, ld w), one warp per (c, l)
        for (int pr = warp; pr < w * ell; pr += nw) {
            const int c = pr % w, l = pr / w;
            const double* uc = U + (int64_t)c * pc.u_ld;
            const double* ql = Qm + (int64_t)l * m + pc.u_row0;
            double d = 0.0;
            for (int i = lane; i < pc.u_rows; i += 32) d += uc[i] * ql[i];
            d = warp_sum(d);
            if (lane == 0) Pp[c + (int64_t)l * w] = pc.alpha * d;
        }
        __syncthreads();
        // W[v_row0 + i, l] += sum_c V[i, c] P_p[c, l]
        for (int i = threadIdx.x; i < pc.v_rows; i += blockDim.x) {
            for (int l0 = 0; l0 < ell; l0 += TR_RB) {
                const int lc = min(TR_RB, ell - l0);
                double acc[TR_RB];
#pragma unroll
                for (int j = 0; j < TR_RB; ++j) acc[j] = 0.0;
                for (int c = 0; c < w; ++c) {
                    const double v = V[i + (int64_t)c * pc.v_ld];
#pragma unroll
                    for (int j = 0; j < TR_RB; ++j)
                        if (j < lc) acc[j] += v * Pp[c + (int64_t)(l0 + j) * w];
                }
                for (int j = 0; j < lc; ++j) Wm[pc.v_row0 + i + (int64_t)(l0 + j) * q] += acc[j];
            }
        }
        __syncthreads();
        flops += 4.0 * (double)ell * w * (pc.u_rows + pc.v_rows);
        bytes += 8.0 * w * (double)(pc.u_rows + pc.v_rows);
    }
    // ---- W = Q_W R;  S = R^T;  one-sided Jacobi S Z = X (orthogonal columns)
    house_qr(Wm, q, ell, tau, scratch);
    const int Kw = min(q, ell);
    for (int idx = threadIdx.x; idx < ell * Kw; idx += blockDim.x) {
        const int i = idx % ell, j = idx / ell;      // S[i][j] = R[j][i] (ell x Kw), R upper
        S[i + (int64_t)j * ell] = (i >= j) ? Wm[j + (int64_t)i * q] : 0.0;
    }
    __syncthreads();
    jacobi_svd(S, ell, Kw, Z, &s_flag);
    for (int j = warp; j < Kw; j += nw) {
        double s = 0.0;
        for (int r = lane; r < ell; r += 32) s += S[r + (int64_t)j * ell] * S[r + (int64_t)j * ell];
        s = warp_sum(s);
        if (lane == 0) sig[j] = sqrt(s);
    }
    __syncthreads();
    const int kk = min(Kw, ORDER_MAX);
    for (int j = threadIdx.x; j < kk; j += blockDim.x) {
        int pos = 0;
        const double sj = sig[j];
        for (int b = 0; b < kk; ++b) pos += (sig[b] > sj || (sig[b] == sj && b < j)) ? 1 : 0;
        order[pos] = j;
    }
    __syncthreads();
    {
        const double smax = sig[order[0]];
        int cnt = 0;
        for (int j = threadIdx.x; j < kk; j += blockDim.x) cnt += (sig[j] > eps * smax && sig[j] > 0.0) ? 1 : 0;
        const double tot = block_sum((double)cnt, scratch);
        if (threadIdx.x == 0) {
            int r = (int)(tot + 0.5);
            if (r > cap) { atomicOr(flags + 1, 2); r = cap; }
            s_rank = r;
        }
    }
    __syncthreads();
    const int r = s_rank;
    // U_out = Q S(:, order)   (m x r);  M^T ~ Q_W R Q^T  =>  M ~ Q R^T Q_W^T = Q (S Z^T) Q_W^T
    double* Uo = pool + t.u_out;
    double* Vo = pool + t.v_out;
    for (int i = threadIdx.x; i < m; i += blockDim.x) {
        for (int c = 0; c < r; ++c) {
            const double* sc = S + (int64_t)order[c] * ell;
            double s = 0.0;
            for (int l = 0; l < ell; ++l) s += Qm[i + (int64_t)l * m] * sc[l];
            Uo[i + (int64_t)c * m] = s;
        }
    }
    // V_out = Q_W [Z(:, order); 0]   (q x r)
    for (int idx = threadIdx.x; idx < q * r; idx += blockDim.x) {
        const int i = idx % q, c = idx / q;
        Vo[i + (int64_t)c * q] = (i < Kw) ? Z[i + (int64_t)order[c] * Kw] : 0.0;
    }
    __syncthreads();
    house_apply_q(Wm, q, Kw, tau, Vo, r);
    if (threadIdx.x == 0) {
        ranks[t.rslot] = r;
        const double el = ell, qd = q, md = m, kw = Kw, rd = r;
        flops += 2.0 * (qd * el * kw - kw * kw * kw / 3.0) + 3.0 * kw * (kw - 1.0) * (el + kw) + 2.0 * md * el * rd +
                 4.0 * qd * kw * rd;
        bytes += 8.0 * rd * (md + qd);
        atomicAdd(ctr + CTR_TRUNC + 0, flops);
        atomicAdd(ctr + CTR_TRUNC + 1, bytes);
    }
}

// dynamic shared memory (bytes) the truncation needs
constexpr int TR_SMEM = (TR_WMAX_SM * TR_RB + TR_LMAX * TR_RB) * 8 + ORDER_MAX * 4;

__device__ __forceinline__ void trunc_run(const TTask& t, const TPiece* __restrict__ pieces, double* pool, int* ranks,
                                          int* flags, double eps, double* ctr, double* dsm) {
    int K = 0;
    for (int p = 0; p < t.piece_count; ++p) K += dim_eval(pieces[t.piece_begin + p].w, ranks);
    if (t.kmax_tot <= TR_EXACT_K) trunc_exact(t, K, pieces, pool, ranks, flags, eps, ctr, dsm);
    else trunc_rand(t, K, pieces, pool, ranks, flags, eps, ctr, dsm);
}

}  // namespace hm
