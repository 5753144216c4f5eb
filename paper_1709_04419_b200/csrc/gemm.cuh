// CTA-level fp64 GEMM on the FP64 tensor cores (mma.sync m8n8k4 f64 -> DMMA):
//
//   C[M x N] = alpha * op(A)[M x Kd] * op(B)[Kd x N] + beta * C      (column-major)
//
// op(A) = A (A is M x Kd, lda) or A^T (A stored Kd x M, lda); likewise op(B).
// Output tiles of BM x BN are distributed over a group of CTAs (tile = first,
// first + step, ...), so one call runs on one CTA or on the nsub CTAs of a
// cooperative truncation.  K chunks of GM_BK are streamed global -> shared
// memory with cp.async (8-byte copies, zero-fill outside the matrix) through a
// GM_NS-stage pipeline, so several chunks are in flight while the DMMAs of the
// current one run.  Three shapes: wide (64 x 64 tiles, warp tile 16 x 32),
// narrow (128 x 16, warp tile 16 x 16) for the probe blocks, and short
// (16 x 128) for transposed probe blocks.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "tile.cuh"

namespace hm {

constexpr int GM_BK = 16;
constexpr int GM_NS = 4;      // stages of the tile-VM products (staged in two 64 x 68 tiles)
#ifndef HM_GM_NSC
#define HM_GM_NSC 4
#endif
#ifndef HM_GM_BKC
#define HM_GM_BKC 16
#endif
constexpr int GM_BKC = HM_GM_BKC;   // K chunk of cta_gemm (truncations); 32 measured no faster
                                    // at n = 64k (the truncations are latency-bound)
constexpr int GM_NSC = HM_GM_NSC;   // stages of cta_gemm (truncations); 8 measured slower at
                                    // n = 64k (the truncation products are short: the ramp counts)

struct GOp {
    const double* p;
    int64_t ld;
    bool trans;
};
__device__ __forceinline__ GOp gop(const double* p, int64_t ld, bool trans) { return GOp{p, ld, trans}; }

// Staged chunk layouts (doubles): an operand whose memory is contiguous along the
// tile dimension (A not transposed, B transposed) is staged [k][i] with ld BM + 4,
// one contiguous along k (A transposed, B not) is staged [i][k] with ld BK + 4.
// Both keep rows 16-byte aligned for 16-byte cp.async and make every DMMA
// fragment load conflict-free per half-warp (bank offsets 8t + 2g resp. 8g + 2t).
template <int BM>
constexpr int gemm_stage_doubles() {
    return (GM_BKC * (BM + 4) > BM * (GM_BKC + 4)) ? GM_BKC * (BM + 4) : BM * (GM_BKC + 4);
}
template <int BM, int BN>
constexpr int gemm_smem_doubles() {
    return GM_NSC * (gemm_stage_doubles<BM>() + gemm_stage_doubles<BN>());
}

__device__ __forceinline__ void cp_async8(double* dst_smem, const double* src, bool valid) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst_smem);
    const int sz = valid ? 8 : 0;                        // 0 -> zero fill
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(src), "r"(sz) : "memory");
}
// 16-byte copy of nbytes (0, 8 or 16) source bytes, the rest zero-filled
__device__ __forceinline__ void cp_async16(double* dst_smem, const double* src, int nbytes) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst_smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(nbytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// Per-thread share of one operand's chunk copies: NP element pairs, each two
// elements adjacent in memory, zero-filled outside the matrix.  VEC: one 16-byte
// cp.async per pair (operand 16-byte aligned with an even ld), else two 8-byte
// copies.  KC: the operand is contiguous along k (staged [row][k]), else along its
// rows (staged [k][row]).  Per tile the pair's pointer and row validity are set;
// per chunk the pointer advances by one chunk of k.  (With a zero source size
// cp.async reads nothing, so the pointer may run past the matrix.)
template <int BD, int NP, bool KC, bool VEC>
struct GCopy {
    const double* ptr[NP];    // element of the pair at the next chunk's k0
    int lim[NP];              // KC: Kd - k if the row is inside, else 0;  !KC: Kd - k
    int nrow[NP];             // !KC: elements of the pair inside along the rows (0..2)
    static constexpr int NPAIR = GM_BKC * BD / 2;

    __device__ __forceinline__ static int row_of(int pr) { return KC ? pr / (GM_BKC / 2) : 2 * (pr % (BD / 2)); }
    __device__ __forceinline__ static int k_of(int pr) { return KC ? 2 * (pr % (GM_BKC / 2)) : pr / (BD / 2); }
    __device__ __forceinline__ static int soff(int pr) {
        return KC ? row_of(pr) * (GM_BKC + 4) + k_of(pr) : k_of(pr) * (BD + 4) + row_of(pr);
    }
    __device__ __forceinline__ void setup(const double* p, int64_t ld, int r0, int R, int Kd) {
#pragma unroll
        for (int e = 0; e < NP; ++e) {
            const int pr = threadIdx.x + e * 256;
            const int r = r0 + row_of(pr), k = k_of(pr);
            ptr[e] = p + (KC ? (int64_t)r * ld + k : r + (int64_t)k * ld);
            lim[e] = (KC && r >= R) ? 0 : Kd - k;
            nrow[e] = KC ? 2 : (r + 1 < R ? 2 : (r < R ? 1 : 0));
        }
    }
    // copies the chunk at k0 (the chunks are issued in order) and advances
    __device__ __forceinline__ void issue(int64_t ld, int k0, double* stage) {
#pragma unroll
        for (int e = 0; e < NP; ++e) {
            const int pr = threadIdx.x + e * 256;
            if (NPAIR % 256 != 0 && pr >= NPAIR) break;
            const int left = lim[e] - k0;
            const int n = KC ? min(max(left, 0), 2) : (left > 0 ? nrow[e] : 0);
            double* dst = stage + soff(pr);
            if (VEC) {
                cp_async16(dst, ptr[e], 8 * n);
            } else {
                cp_async8(dst, ptr[e], n >= 1);
                cp_async8(dst + 1, ptr[e] + 1, n >= 2);
            }
            ptr[e] += KC ? (int64_t)GM_BKC : (int64_t)GM_BKC * ld;
        }
    }
};

// TA / TB: op(A) = A^T / op(B) = B^T (compile time: the staged layouts and fragment
// offsets become constants); the GOp's trans flags must agree (checked).
template <int BM, int BN, int WM, int WN, bool TA, bool TB, bool VA, bool VB>
__device__ void cta_gemm_impl(int M, int N, int Kd, double alpha, const GOp A, const GOp B, double beta, double* C,
                              int64_t ldc, int first, int step, double* smem) {
    static_assert((BM / WM) * (BN / WN) == 8, "8 warps");
    constexpr int FM = WM / 8, FN = WN / 8;              // DMMA blocks per warp
    constexpr int SA = gemm_stage_doubles<BM>(), SB = gemm_stage_doubles<BN>();   // doubles per stage
    constexpr int NPA = (GM_BKC * BM / 2 + 255) / 256, NPB = (GM_BKC * BN / 2 + 255) / 256;
    // A^T is contiguous along k, A along rows; B along k, B^T along columns
    constexpr bool KCA = TA, KCB = !TB;
    // staged strides (doubles) of the tile row and of k for the fragment loads
    constexpr int ARS = KCA ? GM_BKC + 4 : 1, AKS = KCA ? 1 : BM + 4;
    constexpr int BRS = KCB ? GM_BKC + 4 : 1, BKS = KCB ? 1 : BN + 4;
    double* As = smem;                                   // [stage] A chunk
    double* Bs = smem + GM_NSC * SA;                     // [stage] B chunk
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int wm = (warp / (BN / WN)) * WM, wn = (warp % (BN / WN)) * WN;
    const int tm = (M + BM - 1) / BM, tn = (N + BN - 1) / BN;
    const int nk = (Kd + GM_BKC - 1) / GM_BKC;
    const int afo = t * AKS + (wm + g) * ARS, bfo = t * BKS + (wn + g) * BRS;
    GCopy<BM, NPA, KCA, VA> ca;
    GCopy<BN, NPB, KCB, VB> cb;
    for (int tile = first; tile < tm * tn; tile += step) {
        const int i0 = (tile % tm) * BM, j0 = (tile / tm) * BN;
        ca.setup(A.p, A.ld, i0, M, Kd);
        cb.setup(B.p, B.ld, j0, N, Kd);
        double acc[FM][FN][2];
#pragma unroll
        for (int a = 0; a < FM; ++a)
#pragma unroll
            for (int b = 0; b < FN; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
        __syncthreads();                                 // previous tile's readers are done with the stages
#pragma unroll
        for (int s = 0; s < GM_NSC - 1; ++s) {
            if (s < nk) {
                ca.issue(A.ld, s * GM_BKC, As + s * SA);
                cb.issue(B.ld, s * GM_BKC, Bs + s * SB);
            }
            cp_async_commit();
        }
        for (int kc = 0; kc < nk; ++kc) {
            cp_async_wait<GM_NSC - 2>();
            __syncthreads();
            if (kc + GM_NSC - 1 < nk) {
                const int sn = (kc + GM_NSC - 1) % GM_NSC;
                ca.issue(A.ld, (kc + GM_NSC - 1) * GM_BKC, As + sn * SA);
                cb.issue(B.ld, (kc + GM_NSC - 1) * GM_BKC, Bs + sn * SB);
            }
            cp_async_commit();
            const double* as = As + (kc % GM_NSC) * SA + afo;
            const double* bs = Bs + (kc % GM_NSC) * SB + bfo;
#pragma unroll
            for (int kk = 0; kk < GM_BKC; kk += 4) {
                double af[FM], bf[FN];
#pragma unroll
                for (int a = 0; a < FM; ++a) af[a] = as[kk * AKS + a * 8 * ARS];
#pragma unroll
                for (int b = 0; b < FN; ++b) bf[b] = bs[kk * BKS + b * 8 * BRS];
#pragma unroll
                for (int a = 0; a < FM; ++a)
#pragma unroll
                    for (int b = 0; b < FN; ++b) dmma_884(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
            }
        }
        cp_async_wait<0>();
#pragma unroll
        for (int a = 0; a < FM; ++a)
#pragma unroll
            for (int b = 0; b < FN; ++b) {
                const int r = i0 + wm + a * 8 + g;
                const int c = j0 + wn + b * 8 + 2 * t;
                if (r < M) {
                    if (c < N) {
                        double* p = C + r + (int64_t)c * ldc;
                        *p = (beta == 0.0) ? alpha * acc[a][b][0] : beta * *p + alpha * acc[a][b][0];
                    }
                    if (c + 1 < N) {
                        double* p = C + r + (int64_t)(c + 1) * ldc;
                        *p = (beta == 0.0) ? alpha * acc[a][b][1] : beta * *p + alpha * acc[a][b][1];
                    }
                }
            }
    }
    __syncthreads();
}

// 16-byte copies when both operands allow them (the planner's blocks and workspaces are
// 16-byte aligned with even leading dimensions except for odd block sizes)
template <int BM, int BN, int WM, int WN, bool TA, bool TB>
__device__ __forceinline__ void cta_gemm(int M, int N, int Kd, double alpha, const GOp A, const GOp B, double beta,
                                         double* C, int64_t ldc, int first, int step, double* smem) {
    if (A.trans != TA || B.trans != TB) __trap();
    const bool vA = ((reinterpret_cast<uintptr_t>(A.p) & 15) == 0) && ((A.ld & 1) == 0);
    const bool vB = ((reinterpret_cast<uintptr_t>(B.p) & 15) == 0) && ((B.ld & 1) == 0);
    if (vA && vB) cta_gemm_impl<BM, BN, WM, WN, TA, TB, true, true>(M, N, Kd, alpha, A, B, beta, C, ldc, first, step, smem);
    else cta_gemm_impl<BM, BN, WM, WN, TA, TB, false, false>(M, N, Kd, alpha, A, B, beta, C, ldc, first, step, smem);
}

// the shapes used: wide 64 x 64 tiles, narrow 128 x 16 (tall probe blocks), short 16 x 128
// (transposed probes); the operand orientations are template arguments <TA, TB>
template <bool TA, bool TB>
__device__ __forceinline__ void gemm_wide(int M, int N, int Kd, double alpha, const GOp A, const GOp B, double beta,
                                          double* C, int64_t ldc, int first, int step, double* smem) {
    cta_gemm<64, 64, 16, 32, TA, TB>(M, N, Kd, alpha, A, B, beta, C, ldc, first, step, smem);
}
template <bool TA, bool TB>
__device__ __forceinline__ void gemm_narrow(int M, int N, int Kd, double alpha, const GOp A, const GOp B, double beta,
                                            double* C, int64_t ldc, int first, int step, double* smem) {
    cta_gemm<128, 16, 16, 16, TA, TB>(M, N, Kd, alpha, A, B, beta, C, ldc, first, step, smem);
}
template <bool TA, bool TB>
__device__ __forceinline__ void gemm_short(int M, int N, int Kd, double alpha, const GOp A, const GOp B, double beta,
                                           double* C, int64_t ldc, int first, int step, double* smem) {
    cta_gemm<16, 128, 16, 16, TA, TB>(M, N, Kd, alpha, A, B, beta, C, ldc, first, step, smem);
}
__device__ __forceinline__ int gemm_tiles(int M, int N, int bm, int bn) { return ((M + bm - 1) / bm) * ((N + bn - 1) / bn); }

constexpr int GEMM_SMEM_DOUBLES = gemm_smem_doubles<128, 16>() > gemm_smem_doubles<64, 64>()
                                      ? gemm_smem_doubles<128, 16>()
                                      : gemm_smem_doubles<64, 64>();
static_assert(gemm_smem_doubles<16, 128>() <= GEMM_SMEM_DOUBLES, "short shape fits");

}  // namespace hm
