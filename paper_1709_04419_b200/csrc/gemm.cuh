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

template <int BM, int BN>
constexpr int gemm_smem_doubles() {
    return GM_NSC * (GM_BKC * (BM + 1) + GM_BKC * (BN + 1));
}

__device__ __forceinline__ void cp_async8(double* dst_smem, const double* src, bool valid) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst_smem);
    const int sz = valid ? 8 : 0;                        // 0 -> zero fill
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(src), "r"(sz) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

template <int BM, int BN, int WM, int WN>
__device__ void cta_gemm(int M, int N, int Kd, double alpha, const GOp A, const GOp B, double beta, double* C,
                         int64_t ldc, int first, int step, double* smem) {
    static_assert((BM / WM) * (BN / WN) == 8, "8 warps");
    constexpr int FM = WM / 8, FN = WN / 8;              // DMMA blocks per warp
    constexpr int LA = BM + 1, LB = BN + 1;              // padded leading dims of the staged chunks
    constexpr int SA = GM_BKC * LA, SB = GM_BKC * LB;      // doubles per stage
    constexpr int NA = (GM_BKC * BM + 255) / 256, NB = (GM_BKC * BN + 255) / 256;
    double* As = smem;                                   // [stage][k][i]
    double* Bs = smem + GM_NSC * SA;                      // [stage][k][j]
    const bool tA = A.trans, tB = B.trans;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int wm = (warp / (BN / WN)) * WM, wn = (warp % (BN / WN)) * WN;
    const int tm = (M + BM - 1) / BM, tn = (N + BN - 1) / BN;
    const int nk = (Kd + GM_BKC - 1) / GM_BKC;
    for (int tile = first; tile < tm * tn; tile += step) {
        const int i0 = (tile % tm) * BM, j0 = (tile / tm) * BN;
        auto issue = [&](int kc) {                       // chunk kc -> stage kc % NS
            const int k0 = kc * GM_BKC;
            double* as = As + (kc % GM_NSC) * SA;
            double* bs = Bs + (kc % GM_NSC) * SB;
#pragma unroll
            for (int e = 0; e < NA; ++e) {
                const int idx = threadIdx.x + e * 256;
                if (idx < GM_BKC * BM) {
                    int i, k;
                    if (tA) { k = idx % GM_BKC; i = idx / GM_BKC; } else { i = idx % BM; k = idx / BM; }
                    const int gi = i0 + i, gk = k0 + k;
                    const bool ok = gi < M && gk < Kd;
                    cp_async8(as + k * LA + i, ok ? (tA ? A.p + gk + (int64_t)gi * A.ld : A.p + gi + (int64_t)gk * A.ld) : A.p,
                              ok);
                }
            }
#pragma unroll
            for (int e = 0; e < NB; ++e) {
                const int idx = threadIdx.x + e * 256;
                if (idx < GM_BKC * BN) {
                    int j, k;
                    if (tB) { j = idx % BN; k = idx / BN; } else { k = idx % GM_BKC; j = idx / GM_BKC; }
                    const int gj = j0 + j, gk = k0 + k;
                    const bool ok = gj < N && gk < Kd;
                    cp_async8(bs + k * LB + j, ok ? (tB ? B.p + gj + (int64_t)gk * B.ld : B.p + gk + (int64_t)gj * B.ld) : B.p,
                              ok);
                }
            }
        };
        double acc[FM][FN][2];
#pragma unroll
        for (int a = 0; a < FM; ++a)
#pragma unroll
            for (int b = 0; b < FN; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
        __syncthreads();                                 // previous tile's readers are done with the stages
#pragma unroll
        for (int s = 0; s < GM_NSC - 1; ++s) {
            if (s < nk) issue(s);
            cp_async_commit();
        }
        for (int kc = 0; kc < nk; ++kc) {
            cp_async_wait<GM_NSC - 2>();
            __syncthreads();
            if (kc + GM_NSC - 1 < nk) issue(kc + GM_NSC - 1);
            cp_async_commit();
            const double* as = As + (kc % GM_NSC) * SA;
            const double* bs = Bs + (kc % GM_NSC) * SB;
#pragma unroll
            for (int kk = 0; kk < GM_BKC; kk += 4) {
                double af[FM], bf[FN];
#pragma unroll
                for (int a = 0; a < FM; ++a) af[a] = as[(kk + t) * LA + wm + a * 8 + g];
#pragma unroll
                for (int b = 0; b < FN; ++b) bf[b] = bs[(kk + t) * LB + wn + b * 8 + g];
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
