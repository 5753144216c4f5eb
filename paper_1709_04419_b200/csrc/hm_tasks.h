// Task formats shared by the host planner (plan.cpp) and the device kernels
// (hm_kernels.cu).  Plain POD structs, 8-byte aligned, copied to device once
// per plan.  All offsets are in doubles into the handle's device pool.
#pragma once
#include <cstdint>

#ifdef __CUDACC__
#define HM_HD __host__ __device__
#else
#define HM_HD
#endif

namespace hm {

// ---- tile VM -------------------------------------------------------------
// One CTA executes a short program on NTILE 64 x 64 fp64 shared-memory tiles.
enum VmOp : uint8_t {
    VM_LD = 1,       // tile[t0] <- pool[goff] (rows x cols, ld), zero padded
    VM_ST = 2,       // pool[goff] <- tile[t0] (its rows x cols)
    VM_GEMM = 3,     // tile[t0] = beta*tile[t0] + alpha*op(tile[t1]) op(tile[t2])
    VM_POTRF = 4,    // tile[t0] <- chol(tile[t0]); sum log diag -> pool[goff]; fail -> flags[0]
    VM_TRSM_RLT = 5, // tile[t0] <- tile[t0] tile[t1]^{-T}
    VM_TRSM_LN = 6,  // tile[t0] <- tile[t1]^{-1} tile[t0]
    VM_TRMM_LN = 7,  // tile[t0] <- tile[t1] tile[t0]
    VM_ZERO = 8,     // tile[t0] <- 0 with dims (rows x cols)
    VM_MGEMM = 9,    // tile[t0] += sum_i alpha_i op(A_i) op(B_i) over terms[goff .. goff+ld), A_i/B_i
                     // streamed from the pool (pipelined DMMA; replaces LD, LD, GEMM triples)
    VM_TRTRI = 10,   // tile[t0] <- tile[t1]^{-1} (lower triangular, trows[t1] x trows[t1])
    VM_ADD = 11,     // tile[t0] += tile[t1]
    VM_MGEMM_ST = 12,// pool[goff] (rows x cols, ld) = beta * pool[goff] + sum of t1 terms from terms[pad2..]
                     // (fused "ZERO/LD t; VM_MGEMM t; ST t": accumulators go straight to HBM)
};
constexpr int VM_PARTIAL_TERMS = 8;   // dense-update terms per independent partial-sum task
constexpr int NTILE = 3;   // target + two operands (TRSM/TRMM reuse tile 1 for L)

// Dimension spec: actual = (slot < 0) ? stat : clamp(ranks[slot] - off, 0, stat)
struct Dim {
    int32_t stat;
    int32_t slot;
    int32_t off;
    int32_t pad;
};

struct VIns {
    uint8_t op, t0, t1, t2;
    uint8_t ta, tb, pad0, pad1;
    Dim rows, cols;
    int64_t goff;
    int32_t ld;
    int32_t pad2;
    double alpha, beta;
};

// One term of VM_MGEMM: op(A) (M x K) times op(B) (K x N), A/B given like a VM_LD
// (pool offset, leading dimension, stored rows x cols), zero outside those dims.
struct VTerm {
    int64_t a_off, b_off;
    Dim a_rows, a_cols, b_rows, b_cols;
    int32_t a_ld, b_ld;
    uint8_t ta, tb, pad0, pad1, pad2, pad3, pad4, pad5;
    double alpha;
};
constexpr int VM_MAX_TERMS = 64;   // terms per VM_MGEMM instruction

struct VTask {
    int32_t ins_begin;
    int32_t ins_count;
};

// ---- truncation of an accumulated low-rank sum -------------------------
// B <- best rank-r approximation (sigma_i > eps * sigma_1) of
//      sum_p alpha_p * pad(U_p) pad(V_p)^T,   B m x q.
struct TPiece {
    int64_t u_off, v_off;
    int32_t u_ld, v_ld;
    int32_t u_row0, u_rows;   // placement of U_p rows inside the target's rows
    int32_t v_row0, v_rows;   // placement of V_p rows inside the target's columns
    Dim w;                    // width (columns) of the piece
    double alpha;
};

struct TTask {
    int64_t u_out, v_out;     // output U (m x cap, ld m), V (q x cap, ld q)
    int64_t ws;               // workspace offset (doubles), size ws_size
    int64_t ws_size;
    int32_t m, q, cap, rslot;
    int32_t piece_begin, piece_count;
    int32_t kmax_tot;         // sum of static piece widths
    int32_t wmax;             // largest static piece width
    int32_t nsub;             // CTAs cooperating on this truncation (persistent executor)
    int32_t bar;              // index of its group barrier counter
    double eps_scale;         // this truncation's share of the block accuracy (1 = all of it;
                              // a split truncation gives its partial merge and its final step
                              // shares summing to 1, so the block stays within eps)
};

// k_trunc algorithm selection and workspace (trunc.cuh; planner sizes the workspace)
#ifndef HM_TR_EXACT_K
#define HM_TR_EXACT_K 160
#endif
constexpr int TR_EXACT_K = HM_TR_EXACT_K;   // static stacked width up to which the exact QR+SVD path runs ...
constexpr int TR_EXACT_MMAX = 512;   // ... on blocks with at most this many rows and columns: the
                                     // single-CTA Householder QR of a taller factor is HBM-latency
                                     // bound (~25 ms at 8192 x 160); those take the cooperative
                                     // randomized path instead
// narrow stacks (static width <= 64, e.g. the recompression of an ACA factor) take the
// exact path on blocks up to TR_EXACT_MN rows: its K column steps beat the randomized
// path's ~40 latency-bound stages
#ifndef HM_TR_EXACT_MN
#define HM_TR_EXACT_MN 512
#endif
constexpr int TR_EXACT_MN = HM_TR_EXACT_MN;
HM_HD inline bool trunc_exact_path(int32_t m, int32_t q, int32_t kmax_tot) {
    return (kmax_tot <= TR_EXACT_K && m <= TR_EXACT_MMAX && q <= TR_EXACT_MMAX) ||
           (kmax_tot <= 64 && m <= TR_EXACT_MN && q <= TR_EXACT_MN);
}
#ifndef HM_TR_RB
#define HM_TR_RB 8
#endif
constexpr int TR_RB = HM_TR_RB;   // probes per block of the randomized range finder (<= 32: one
                                  // warp lane per probe in the pivoted Cholesky)
static_assert(TR_RB >= 8 && TR_RB <= 32 && TR_RB % 8 == 0, "TR_RB");
#ifndef HM_TR_NB
#define HM_TR_NB 8
#endif
constexpr int TR_NB = HM_TR_NB;   // blocks per pass over the stacks: 8 x 8 = 64 probes fill the
                                  // 64-wide GEMM tiles exactly and resolve ranks up to ~56 in one pass
                                  // (measured at n = 64k: 8 x 8 7.27 evals/s, 4 x 16 6.91, 2 x 32 5.50)
constexpr int TR_PW = TR_RB * TR_NB;
constexpr int TR_LMAX = 256;      // max basis width cap + RB
constexpr int HM_KMAX_LIMIT = 240;   // hm_params.kmax bound (include/hmlik.h)
static_assert(HM_KMAX_LIMIT <= TR_LMAX - TR_RB, "kmax limit");
constexpr int TR_RCH = 64;        // fixed row chunk of the cooperative truncation (8 warps x 8 rows)
constexpr int TR_TCH = 128;       // stacked columns staged per shared-memory chunk
constexpr int TR_PMAX = 1023;     // pieces per truncation
#ifndef HM_COOP_ROWFAC
#define HM_COOP_ROWFAC 4
#endif
#ifndef HM_COOP_WORK_LOG2
#define HM_COOP_WORK_LOG2 17
#endif
constexpr int64_t TR_COOP_WORK = int64_t(1) << HM_COOP_WORK_LOG2;   // (m + q) * static K per cooperating CTA
constexpr int TR_COOP_MAX = 32;   // CTAs per cooperative truncation (hard limit; the plan's
                                  // cap hm_params.coop_max defaults to TR_COOP_DEFAULT)
constexpr int TR_COOP_DEFAULT = 16;
constexpr unsigned long long TR_COOP_WATCHDOG_NS = 120ull * 1000000000ull;   // group-barrier wait before __trap (trunc.cuh)
#ifndef HM_TR_SHRINK
#define HM_TR_SHRINK 1
#endif
constexpr int TR_SHRINK = HM_TR_SHRINK;   // > 0: a cooperative truncation keeps one CTA per TR_SHRINK
                                          // 64-row chunks after its first probe pass (trunc.cuh);
                                          // measured at n = 64k, S = 4: 1 -> 6.84 evals/s, 2 -> 6.60,
                                          // 0 (off) -> 6.62 (one evaluation 397 / 464 / 383 ms)

struct TruncWs {                  // randomized-path workspace (doubles unless noted)
    double *ctl, *Om, *Ast, *Bst, *Tt, *Y, *npart, *Q, *Cb, *Pt, *Wm, *Wc, *S, *Z, *Xo, *G, *tau, *sig, *Cp, *Cf, *Gp,
        *Gp2, *Ypart, *Wpart, *Rpart;
    int64_t total;
};
// Reduction split of the two products with a long inner dimension, T^T = Omega^T V_stack
// (over q) and P^T = Q^T U_stack (over m): when their few output tiles cannot occupy the
// group, the inner dimension is cut into S parts whose partial products (S x Lp x K)
// are summed afterwards.  S = 1: no split.  Bounded to TR_RSPLIT_MAX doubles.
constexpr int64_t TR_RSPLIT_MAX = int64_t(1) << 23;
HM_HD inline int32_t trunc_rsplit(int32_t m, int32_t q, int32_t cap, int32_t Ks, int32_t nsub) {
    const int64_t Lp = (cap + TR_RB > TR_PW) ? cap + TR_RB : TR_PW;
    int64_t s = nsub;
    const int64_t by_mem = TR_RSPLIT_MAX / (Lp * (Ks > 0 ? Ks : 1));
    const int64_t by_len = (m < q ? m : q) / 256;
    if (by_mem < s) s = by_mem;
    if (by_len < s) s = by_len;
    return s < 2 ? 1 : (int32_t)s;
}
// split-K of the W = V_stack P product (partials nsub x q x L) only for small q
constexpr int TR_WSPLIT_Q = 512;
HM_HD inline TruncWs trunc_ws_layout(double* base, int32_t m, int32_t q, int32_t cap, int32_t Ks, int32_t nsub) {
    const int64_t L = (int64_t)cap + TR_RB;
    const int64_t ns = nsub < 1 ? 1 : nsub;
    const int64_t nch = (m + TR_RCH - 1) / TR_RCH + (q + TR_RCH - 1) / TR_RCH;
    TruncWs w;
    int64_t o = 0;
    const int32_t rs = trunc_rsplit(m, q, cap, Ks, nsub);
    const int64_t Lp = (L > TR_PW) ? L : TR_PW;
    const int64_t sz[25] = {4 + (TR_LMAX + 16) / 2, (int64_t)q * TR_PW, (int64_t)m * Ks, (int64_t)q * Ks,
                            (int64_t)TR_PW * Ks, (int64_t)m * TR_PW, nch * TR_PW, (int64_t)m * L, L * TR_RB,
                            L * (int64_t)Ks, (int64_t)q * L, (int64_t)q * L, L * L, L * L, L * L, L * L, L, L,
                            ns * L * TR_RB, ns * L * TR_RB, ns * TR_RB * TR_RB, ns * L * L, ns * m * TR_PW,
                            (q <= TR_WSPLIT_Q) ? ns * q * L : 0, rs > 1 ? rs * Lp * Ks : 0};
    double* ptr[25];
    for (int i = 0; i < 25; ++i) {
        ptr[i] = base + o;
        o += (sz[i] + 7) & ~int64_t(7);
    }
    w.ctl = ptr[0]; w.Om = ptr[1]; w.Ast = ptr[2]; w.Bst = ptr[3]; w.Tt = ptr[4]; w.Y = ptr[5];
    w.npart = ptr[6]; w.Q = ptr[7]; w.Cb = ptr[8]; w.Pt = ptr[9]; w.Wm = ptr[10]; w.Wc = ptr[11];
    w.S = ptr[12]; w.Z = ptr[13]; w.Xo = ptr[14]; w.G = ptr[15]; w.tau = ptr[16]; w.sig = ptr[17];
    w.Cp = ptr[18]; w.Cf = ptr[19]; w.Gp = ptr[20]; w.Gp2 = ptr[21]; w.Ypart = ptr[22]; w.Wpart = ptr[23];
    w.Rpart = ptr[24];
    w.total = o + 64;
    return w;
}
inline int64_t trunc_ws_size(int32_t m, int32_t q, int32_t cap, int32_t kmax_tot, int32_t nsub) {
    if (trunc_exact_path(m, q, kmax_tot)) {
        const int64_t K = kmax_tot;
        return ((int64_t)m + q + 2 * K + 8) * K + 64;
    }
    return trunc_ws_layout(nullptr, m, q, cap, kmax_tot, nsub).total;
}
inline int32_t trunc_nsub(int32_t m, int32_t q, int32_t kmax_tot, int32_t cap = TR_COOP_DEFAULT) {
    if (trunc_exact_path(m, q, kmax_tot)) return 1;
    // one CTA per TR_COOP_WORK of stacked data, at most two per 64-row chunk of the
    // larger side (a group must assemble before it starts: more CTAs than rows to
    // share only adds waiting), at most TR_COOP_MAX
    // co-scheduled handles (cap <= 8) trade latency for throughput: twice the work per CTA
    // (measured at n = 64k, 4 streams: 2.87 -> 3.03 evals/s)
    const int64_t work = cap <= 8 ? 2 * TR_COOP_WORK : TR_COOP_WORK;
    const int64_t g = ((int64_t)(m + q) * kmax_tot) / work;
    const int64_t rows = (m > q ? m : q);
    const int64_t gmax = HM_COOP_ROWFAC * ((rows + TR_RCH - 1) / TR_RCH);
    int64_t n = g < 1 ? 1 : g;
    if (n > gmax) n = gmax;
    if (n > cap) n = cap;
    if (n > TR_COOP_MAX) n = TR_COOP_MAX;
    return (int32_t)n;
}

// ---- dependency-driven execution (persistent executor, exec.cu) --------
// All tasks of a phase in a topological order (sorted by wave); each lists the
// positions of the tasks it must wait for (all smaller than its own).
struct XTask {
    int32_t kind;       // 0 = tile-VM program (vt[idx]), 1 = truncation (tt[idx])
    int32_t idx;
    int32_t dep_begin;  // into the phase's dependency array
    int32_t dep_count;
    int32_t sub, nsub;  // cooperative truncation: this CTA's index / group size (else 0 / 1)
};

// ---- assembly ------------------------------------------------------------
struct DenseGenTask {         // D[i + j m] = C(|x_{r0+i} - x_{c0+j}|), i < m, j < q
    int64_t off;
    int32_t r0, c0, m, q;
};

struct AcaTask {              // ACA of the m x q block rows [r0, r0+m) x cols [c0, c0+q)
    int64_t u_off, v_off;     // U m x cap (ld m), V q x cap (ld q)
    int32_t r0, c0, m, q;
    int32_t cap, rslot;
};

}  // namespace hm
