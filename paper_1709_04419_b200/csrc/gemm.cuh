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

// One operand's share of a chunk copy: NP element pairs per thread, each pair two
// elements adjacent in memory (one 16-byte cp.async when the operand is 16-byte
// aligned with an even ld, else two 8-byte copies); elements outside the matrix
// are zero-filled.  Operand rows [r0, r0 + BD) of R, contiguous along k when kc.
template <int BD, int NP>
__device__ __forceinline__ void gemm_issue(const double* p, int64_t ld, bool kc, bool vec, int r0, int R, int k0, int Kd,
                                           double* stage) {
#pragma unroll
    for (int e = 0; e < NP; ++e) {
        const int pr = threadIdx.x + e * 256;
        if (pr >= GM_BKC * BD / 2) break;
        int r, k, so, n;   // n: valid elements of the pair
        if (kc) {
            k = 2 * (pr % (GM_BKC / 2)); r = pr / (GM_BKC / 2); so = r * (GM_BKC + 4) + k;
            const int gk = k0 + k;
            n = (r0 + r >= R) ? 0 : (gk + 1 < Kd ? 2 : (gk < Kd ? 1 : 0));
        } else {
            r = 2 * (pr % (BD / 2)); k = pr / (BD / 2); so = k * (BD + 4) + r;
            const int gr = r0 + r;
            n = (k0 + k >= Kd) ? 0 : (gr + 1 < R ? 2 : (gr < R ? 1 : 0));
        }
        const double* src = n ? p + (kc ? (int64_t)(r0 + r) * ld + (k0 + k) : (r0 + r) + (int64_t)(k0 + k) * ld) : p;
        if (vec) {
            cp_async16(stage + so, src, 8 * n);
        } else {
            cp_async8(stage + so, src, n >= 1);
            cp_async8(stage + so + 1, n >= 2 ? src + 1 : p, n >= 2);
        }
    }
}

template <int BM, int BN, int WM, int WN>
__device__ void cta_gemm(int M, int N, int Kd, double alpha, const GOp A, const GOp B, double beta, double* C,
                         int64_t ldc, int first, int step, double* smem) {
    static_assert((BM / WM) * (BN / WN) == 8, "8 warps");
    constexpr int FM = WM / 8, FN = WN / 8;              // DMMA blocks per warp
    constexpr int SA = gemm_stage_doubles<BM>(), SB = gemm_stage_doubles<BN>();   // doubles per stage
    constexpr int NPA = (GM_BKC * BM / 2 + 255) / 256, NPB = (GM_BKC * BN / 2 + 255) / 256;
    double* As = smem;                                   // [stage] A chunk
    double* Bs = smem + GM_NSC * SA;                     // [stage] B chunk
    // A^T is contiguous along k, A along rows; B along k, B^T along columns
    const bool kcA = A.trans, kcB = !B.trans;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int wm = (warp / (BN / WN)) * WM, wn = (warp % (BN / WN)) * WN;
    const int tm = (M + BM - 1) / BM, tn = (N + BN - 1) / BN;
    const int nk = (Kd + GM_BKC - 1) / GM_BKC;
    // staged strides (doubles) of the tile row and of k for the fragment loads
    const int ars = kcA ? GM_BKC + 4 : 1, aks = kcA ? 1 : BM + 4;
    const int brs = kcB ? GM_BKC + 4 : 1, bks = kcB ? 1 : BN + 4;
    const int afo = t * aks + (wm + g) * ars, bfo = t * bks + (wn + g) * brs;
    const bool vA = ((reinterpret_cast<uintptr_t>(A.p) & 15) == 0) && ((A.ld & 1) == 0);
    const bool vB = ((reinterpret_cast<uintptr_t>(B.p) & 15) == 0) && ((B.ld & 1) == 0);
    for (int tile = first; tile < tm * tn; tile += step) {
        const int i0 = (tile % tm) * BM, j0 = (tile / tm) * BN;
        double acc[FM][FN][2];
#pragma unroll
        for (int a = 0; a < FM; ++a)
#pragma unroll
            for (int b = 0; b < FN; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
        __syncthreads();                                 // previous tile's readers are done with the stages
#pragma unroll
        for (int s = 0; s < GM_NSC - 1; ++s) {
            if (s < nk) {
                gemm_issue<BM, NPA>(A.p, A.ld, kcA, vA, i0, M, s * GM_BKC, Kd, As + s * SA);
                gemm_issue<BN, NPB>(B.p, B.ld, kcB, vB, j0, N, s * GM_BKC, Kd, Bs + s * SB);
            }
            cp_async_commit();
        }
        for (int kc = 0; kc < nk; ++kc) {
            cp_async_wait<GM_NSC - 2>();
            __syncthreads();
            if (kc + GM_NSC - 1 < nk) {
                const int sn = (kc + GM_NSC - 1) % GM_NSC;
                gemm_issue<BM, NPA>(A.p, A.ld, kcA, vA, i0, M, (kc + GM_NSC - 1) * GM_BKC, Kd, As + sn * SA);
                gemm_issue<BN, NPB>(B.p, B.ld, kcB, vB, j0, N, (kc + GM_NSC - 1) * GM_BKC, Kd, Bs + sn * SB);
            }
            cp_async_commit();
            const double* as = As + (kc % GM_NSC) * SA + afo;
            const double* bs = Bs + (kc % GM_NSC) * SB + bfo;
#pragma unroll
            for (int kk = 0; kk < GM_BKC; kk += 4) {
                double af[FM], bf[FN];
#pragma unroll
                for (int a = 0; a < FM; ++a) af[a] = as[kk * aks + a * 8 * ars];
#pragma unroll
                for (int b = 0; b < FN; ++b) bf[b] = bs[kk * bks + b * 8 * brs];
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

// the shapes used: wide 64 x 64 tiles, narrow 128 x 16 (tall probe blocks), short 16 x 128 (transposed probes)
__device__ __forceinline__ void gemm_wide(int M, int N, int Kd, double alpha, const GOp A, const GOp B, double beta,
                                          double* C, int64_t ldc, int first, int step, double* smem) {
    cta_gemm<64, 64, 16, 32>(M, N, Kd, alpha, A, B, beta, C, ldc, first, step, smem);
}
__device__ __forceinline__ void gemm_narrow(int M, int N, int Kd, double alpha, const GOp A, const GOp B, double beta,
                                            double* C, int64_t ldc, int first, int step, double* smem) {
    cta_gemm<128, 16, 16, 16>(M, N, Kd, alpha, A, B, beta, C, ldc, first, step, smem);
}
__device__ __forceinline__ void gemm_narrow64(int M, int N, int Kd, double alpha, const GOp A, const GOp B, double beta,
                                              double* C, int64_t ldc, int first, int step, double* smem) {
    cta_gemm<64, 16, 8, 16>(M, N, Kd, alpha, A, B, beta, C, ldc, first, step, smem);
}
__device__ __forceinline__ void gemm_short(int M, int N, int Kd, double alpha, const GOp A, const GOp B, double beta,
                                           double* C, int64_t ldc, int first, int step, double* smem) {
    cta_gemm<16, 128, 16, 16>(M, N, Kd, alpha, A, B, beta, C, ldc, first, step, smem);
}
__device__ __forceinline__ int gemm_tiles(int M, int N, int bm, int bn) { return ((M + bm - 1) / bm) * ((N + bn - 1) / bn); }

constexpr int GEMM_SMEM_DOUBLES = gemm_smem_doubles<128, 16>() > gemm_smem_doubles<64, 64>()
                                      ? gemm_smem_doubles<128, 16>()
                                      : gemm_smem_doubles<64, 64>();
static_assert(gemm_smem_doubles<16, 128>() <= GEMM_SMEM_DOUBLES, "short shape fits");

}  // namespace hm
