// 64 x 64 fp64 shared-memory tile primitives shared by the dense check path
// and the H-Cholesky tile VM.  Tiles are column-major with leading dimension
// TLD = 68 doubles (the +4 pad makes every DMMA m8n8k4 fragment access below
// hit each 8-byte bank pair exactly twice, i.e. two wavefronts per warp load),
// and are kept ZERO outside their logical (rows, cols), so products can run
// over whole k-steps of 4 without masks.
//
// The contraction uses the FP64 tensor-core MMA (mma.sync m8n8k4 .f64 -> SASS
// DMMA); fragment layout (PTX ISA, "Matrix fragments for mma.m8n8k4 with
// .f64"): g = lane>>2, t = lane&3;  A(8x4): a0 = A[g][t];  B(4x8): b0 = B[t][g];
// C(8x8): c0 = C[g][2t], c1 = C[g][2t+1].
#pragma once
#include <cuda_runtime.h>

namespace hm {

constexpr int TD = 64;             // tile dimension
constexpr int TLD = 68;            // tile leading dimension (doubles)
constexpr int TSZ = TD * TLD;      // doubles per tile
constexpr int TTHREADS = 256;      // threads per CTA using tile primitives

__host__ __device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }

__device__ __forceinline__ void dmma_884(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// element accessors for op(A)[r][k] where A is a col-major tile
__device__ __forceinline__ double opA(const double* A, bool tA, int r, int k) {
    return tA ? A[r * TLD + k] : A[k * TLD + r];
}
// op(B)[k][c]
__device__ __forceinline__ double opB(const double* B, bool tB, int k, int c) {
    return tB ? B[k * TLD + c] : B[c * TLD + k];
}

// C = beta*C + alpha*op(A) op(B); C m x n, op(A) m x k, op(B) k x n; all <= 64.
// Must be called by all TTHREADS threads of the CTA; ends with __syncthreads.
// C must not alias A or B.
__device__ __forceinline__ void tile_gemm(double* C, const double* A, bool tA, const double* B, bool tB,
                                          int m, int n, int k, double alpha, double beta) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t = lane & 3;
    const int wr = (warp >> 2) * 32;      // warp row base: 0 or 32
    const int wc = (warp & 3) * 16;       // warp col base: 0,16,32,48
    const bool active = (wr < m) && (wc < n);
    if (active) {
        double acc[4][2][2];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
        const int kk = (k + 3) & ~3;
        const int mi = min(4, (m - wr + 7) >> 3);
        const int nj = min(2, (n - wc + 7) >> 3);
        for (int k0 = 0; k0 < kk; k0 += 4) {
            double a[4], b[2];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = (i < mi) ? opA(A, tA, wr + i * 8 + g, k0 + t) : 0.0;
#pragma unroll
            for (int j = 0; j < 2; ++j) b[j] = (j < nj) ? opB(B, tB, k0 + t, wc + j * 8 + g) : 0.0;
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 2; ++j)
                    if (i < mi && j < nj) dmma_884(acc[i][j][0], acc[i][j][1], a[i], b[j]);
        }
        __syncwarp();
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                if (i < mi && j < nj) {
                    const int r = wr + i * 8 + g;
                    const int c = wc + j * 8 + 2 * t;
                    double* p0 = C + c * TLD + r;
                    double* p1 = C + (c + 1) * TLD + r;
                    if (beta == 0.0) {
                        *p0 = alpha * acc[i][j][0];
                        *p1 = alpha * acc[i][j][1];
                    } else {
                        *p0 = beta * *p0 + alpha * acc[i][j][0];
                        *p1 = beta * *p1 + alpha * acc[i][j][1];
                    }
                }
            }
    }
    __syncthreads();
}

// Zero a whole tile.
__device__ __forceinline__ void tile_zero(double* T) {
    for (int i = threadIdx.x; i < TSZ; i += blockDim.x) T[i] = 0.0;
}

// Load rows x cols (col-major, leading dim ld) from global into a zero-padded tile.
// (ld.global.cg: the source may have been written by another CTA of the same
// persistent kernel, so the read-only / L1 paths are not used)
// All 16 loads of a thread are issued before the first store to shared memory, so a
// tile costs one global-memory latency, not sixteen (TTHREADS = 256 threads).
__device__ __forceinline__ void tile_load(double* T, const double* G, int64_t ld, int rows, int cols) {
    if (blockDim.x == TTHREADS) {
        constexpr int PER = TD * TD / TTHREADS;
        double v[PER];
#pragma unroll
        for (int u = 0; u < PER; ++u) {
            const int idx = threadIdx.x + u * TTHREADS;
            const int r = idx & (TD - 1), c = idx >> 6;
            v[u] = (r < rows && c < cols) ? __ldcg(G + (int64_t)c * ld + r) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < PER; ++u) {
            const int idx = threadIdx.x + u * TTHREADS;
            T[(idx >> 6) * TLD + (idx & (TD - 1))] = v[u];
        }
        return;
    }
    for (int idx = threadIdx.x; idx < TD * TD; idx += blockDim.x) {
        const int r = idx & (TD - 1), c = idx >> 6;
        T[c * TLD + r] = (r < rows && c < cols) ? __ldcg(G + (int64_t)c * ld + r) : 0.0;
    }
}

__device__ __forceinline__ void tile_store(const double* T, double* __restrict__ G, int64_t ld, int rows, int cols) {
    for (int idx = threadIdx.x; idx < TD * TD; idx += blockDim.x) {
        const int r = idx & (TD - 1), c = idx >> 6;
        if (r < rows && c < cols) G[(int64_t)c * ld + r] = T[c * TLD + r];
    }
}

// In-place lower Cholesky of the m x m tile A (upper part ignored and zeroed).
// Returns (to all threads) the number of failed pivots (0 on success); on
// failure the offending pivot is replaced by 1 so the factor stays finite.
// *logdiag_sum receives sum_i log A_ii of the factor (thread 0).
// Left-looking by columns (the Cholesky is on the factorisation's critical path:
// latency matters, not flops): for column j, a group of 4 lanes per row i >= j
// forms A_ij - sum_{k<j} L_ik L_jk (strided over k, shuffle-reduced); then the
// pivot and the scaling.  Two CTA barriers per column.  Needs blockDim.x = 256.
__device__ __forceinline__ int tile_potrf(double* A, int m, double* logdiag_sum) {
    __shared__ int s_fail;
    __shared__ double s_v[TD];
    const int r = threadIdx.x >> 2, p = threadIdx.x & 3;
    if (threadIdx.x == 0) s_fail = 0;
    for (int j = 0; j < m; ++j) {
        double sum = 0.0;
        const bool act = r >= j && r < m;
        if (act)
            for (int k = p; k < j; k += 4) sum += A[k * TLD + r] * A[k * TLD + j];
        sum += __shfl_xor_sync(0xffffffffu, sum, 1);
        sum += __shfl_xor_sync(0xffffffffu, sum, 2);
        if (act && p == 0) s_v[r] = A[j * TLD + r] - sum;
        __syncthreads();
        if (act && p == 0) {
            const double d = s_v[j];
            const double piv = (d > 0.0) ? sqrt(d) : 1.0;
            if (r == j) {
                A[j * TLD + j] = piv;
                if (!(d > 0.0)) s_fail += 1;
            } else {
                A[j * TLD + r] = s_v[r] / piv;
            }
        }
        __syncthreads();
    }
    // zero the strict upper triangle
    for (int idx = threadIdx.x; idx < m * m; idx += blockDim.x) {
        const int i = idx % m, c = idx / m;
        if (c > i) A[c * TLD + i] = 0.0;
    }
    if (logdiag_sum != nullptr && threadIdx.x < 32) {
        double s = 0.0;
        for (int j = threadIdx.x; j < m; j += 32) s += log(A[j * TLD + j]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (threadIdx.x == 0) *logdiag_sum = s;
    }
    __syncthreads();
    return s_fail;
}

// B <- B L^{-T}: B m x p, L p x p lower (solves X L^T = B row by row).
__device__ __forceinline__ void tile_trsm_rlt(double* B, const double* L, int m, int p) {
    for (int r = threadIdx.x; r < m; r += blockDim.x) {
        for (int c = 0; c < p; ++c) {
            double s = B[c * TLD + r];
            for (int k = 0; k < c; ++k) s -= B[k * TLD + r] * L[k * TLD + c];
            B[c * TLD + r] = s / L[c * TLD + c];
        }
    }
    __syncthreads();
}

// B <- L^{-1} B: L m x m lower, B m x k (forward substitution per column).
__device__ __forceinline__ void tile_trsm_ln(double* B, const double* L, int m, int k) {
    for (int c = threadIdx.x; c < k; c += blockDim.x) {
        for (int r = 0; r < m; ++r) {
            double s = B[c * TLD + r];
            for (int i = 0; i < r; ++i) s -= L[i * TLD + r] * B[c * TLD + i];
            B[c * TLD + r] = s / L[r * TLD + r];
        }
    }
    __syncthreads();
}

// B <- L B: L m x m lower, B m x k (in place, bottom row first).
__device__ __forceinline__ void tile_trmm_ln(double* B, const double* L, int m, int k) {
    for (int c = threadIdx.x; c < k; c += blockDim.x) {
        for (int r = m - 1; r >= 0; --r) {
            double s = 0.0;
            for (int i = 0; i <= r; ++i) s += L[i * TLD + r] * B[c * TLD + i];
            B[c * TLD + r] = s;
        }
    }
    __syncthreads();
}

// A += B over the whole tile (both zero outside their logical dims)
__device__ __forceinline__ void tile_add(double* A, const double* B) {
    for (int i = threadIdx.x; i < TSZ; i += blockDim.x) A[i] += B[i];
    __syncthreads();
}

// X <- L^{-1} for the m x m lower-triangular tile L (X lower, zero elsewhere).  Column j
// of X solves L x = e_j by forward substitution; each column is owned by a group of 4
// lanes of one warp (dot products strided over k, shuffle-reduced), so the row-by-row
// dependency stays inside the group: no CTA barrier until the end.  X != L;
// needs blockDim.x = 256.
__device__ __forceinline__ void tile_trtri(double* X, const double* L, int m) {
    tile_zero(X);
    __syncthreads();
    const int j = threadIdx.x >> 2, p = threadIdx.x & 3;
    const bool act = j < m;
    if (act && p == 0) X[j * TLD + j] = 1.0 / L[j * TLD + j];
    __syncwarp();
    for (int i = 1; i < m; ++i) {
        double sum = 0.0;
        if (act && i > j)
            for (int k = j + p; k < i; k += 4) sum += L[k * TLD + i] * X[j * TLD + k];
        sum += __shfl_xor_sync(0xffffffffu, sum, 1);
        sum += __shfl_xor_sync(0xffffffffu, sum, 2);
        if (act && i > j && p == 0) X[j * TLD + i] = -sum / L[i * TLD + i];
        __syncwarp();
    }
    __syncthreads();
}

}  // namespace hm
