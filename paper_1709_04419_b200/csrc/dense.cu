// Dense fp64 check path (n <= HM_DENSE_NMAX): exact Eq. (1) on the GPU.
//
//   assemble C(theta) (lower triangle, Eq. 2 via matern_dev)
//   -> blocked right-looking Cholesky C = L L^T with 64 x 64 tiles
//      (tile POTRF, panel TRSM, trailing SYRK on the FP64 tensor cores)
//   -> log det = 2 sum log L_ii (l.283), v = L^{-1} Z (l.265), quad = v^T v.
//
// This path exists to check the H-matrix path against an exact GPU result
// (north star: 1e-10 relative vs the oracle) and as a dense baseline; it is
// not used by the H path.
#include <cuda_runtime.h>

#include <cmath>
#include <vector>

#include "common.h"
#include "dense.h"
#include "matern.cuh"
#include "tile.cuh"

namespace hm {

namespace {

// Lower-triangle tiles of A (n x n col-major) from points (original order, n x 2 row-major).
__global__ void k_dense_matern(double* __restrict__ A, int64_t n, const double* __restrict__ pts, MaternParams p) {
    const int64_t j = (int64_t)blockIdx.y * 16 + threadIdx.y;
    const int64_t i = (int64_t)blockIdx.x * 16 + threadIdx.x;
    if (i >= n || j >= n || i < j) return;
    const double h = dist2d(pts[2 * i], pts[2 * i + 1], pts[2 * j], pts[2 * j + 1]);
    A[j * n + i] = (i == j) ? p.sigma2 : matern_dev(h, p);
}

__global__ void __launch_bounds__(TTHREADS) k_potrf_diag(double* A, int64_t n, int64_t j0, double* logd, int* fail) {
    extern __shared__ double sm[];
    const int m = (int)imin64(TD, n - j0);
    double* T = sm;
    double* Ajj = A + j0 * n + j0;
    tile_load(T, Ajj, n, m, m);
    __syncthreads();
    __shared__ double s_log;
    const int f = tile_potrf(T, m, &s_log);
    tile_store(T, Ajj, n, m, m);
    if (threadIdx.x == 0) {
        logd[j0 / TD] = s_log;
        if (f) atomicAdd(fail, f);
    }
}

__global__ void __launch_bounds__(TTHREADS) k_trsm_panel(double* A, int64_t n, int64_t j0) {
    extern __shared__ double sm[];
    double* L = sm;
    double* B = sm + TSZ;
    const int p = (int)imin64(TD, n - j0);
    const int64_t i0 = j0 + TD + (int64_t)blockIdx.x * TD;
    if (i0 >= n) return;
    const int m = (int)imin64(TD, n - i0);
    tile_load(L, A + j0 * n + j0, n, p, p);
    tile_load(B, A + j0 * n + i0, n, m, p);
    __syncthreads();
    tile_trsm_rlt(B, L, m, p);
    tile_store(B, A + j0 * n + i0, n, m, p);
}

__global__ void __launch_bounds__(TTHREADS) k_syrk_trailing(double* A, int64_t n, int64_t j0) {
    extern __shared__ double sm[];
    double* Ta = sm;
    double* Tb = sm + TSZ;
    double* Tc = sm + 2 * TSZ;
    const int64_t b = blockIdx.x;
    const int64_t I = (int64_t)((sqrt(8.0 * (double)b + 1.0) - 1.0) * 0.5);
    int64_t II = I;
    while ((II + 1) * (II + 2) / 2 <= b) ++II;
    while (II * (II + 1) / 2 > b) --II;
    const int64_t K = b - II * (II + 1) / 2;
    const int64_t base = j0 + TD;
    const int64_t i0 = base + II * TD, k0 = base + K * TD;
    if (i0 >= n || k0 >= n) return;
    const int p = (int)imin64(TD, n - j0);
    const int mi = (int)imin64(TD, n - i0);
    const int mk = (int)imin64(TD, n - k0);
    tile_load(Ta, A + j0 * n + i0, n, mi, p);
    tile_load(Tb, A + j0 * n + k0, n, mk, p);
    tile_load(Tc, A + k0 * n + i0, n, mi, mk);
    __syncthreads();
    tile_gemm(Tc, Ta, false, Tb, true, mi, mk, p, -1.0, 1.0);
    tile_store(Tc, A + k0 * n + i0, n, mi, mk);
}

// Z_j <- L_jj^{-1} Z_j for the column block [c0, c0+kc) of Z (n x k col-major)
__global__ void __launch_bounds__(TTHREADS) k_trsv_diag(const double* A, int64_t n, double* Z, int64_t j0, int kc) {
    extern __shared__ double sm[];
    double* L = sm;
    double* B = sm + TSZ;
    const int64_t c0 = (int64_t)blockIdx.x * TD;
    const int m = (int)imin64(TD, n - j0);
    const int w = (int)imin64(TD, kc - c0);
    tile_load(L, A + j0 * n + j0, n, m, m);
    tile_load(B, Z + c0 * n + j0, n, m, w);
    __syncthreads();
    tile_trsm_ln(B, L, m, w);
    tile_store(B, Z + c0 * n + j0, n, m, w);
}

// Z_i -= L_ij Z_j for all row blocks i > j (grid.x = row block, grid.y = column block)
__global__ void __launch_bounds__(TTHREADS) k_solve_update(const double* A, int64_t n, double* Z, int64_t j0, int kc) {
    extern __shared__ double sm[];
    double* Ta = sm;
    double* Tb = sm + TSZ;
    double* Tc = sm + 2 * TSZ;
    const int64_t i0 = j0 + TD + (int64_t)blockIdx.x * TD;
    const int64_t c0 = (int64_t)blockIdx.y * TD;
    if (i0 >= n) return;
    const int p = (int)imin64(TD, n - j0);
    const int m = (int)imin64(TD, n - i0);
    const int w = (int)imin64(TD, kc - c0);
    tile_load(Ta, A + j0 * n + i0, n, m, p);
    tile_load(Tb, Z + c0 * n + j0, n, p, w);
    tile_load(Tc, Z + c0 * n + i0, n, m, w);
    __syncthreads();
    tile_gemm(Tc, Ta, false, Tb, false, m, w, p, -1.0, 1.0);
    tile_store(Tc, Z + c0 * n + i0, n, m, w);
}

// out[3j+0..2] for column j: (loglik, logdet, quad) -- single CTA reduction.
__global__ void k_dense_finish(const double* logd, int64_t nblk, const double* Z, int64_t n, int k, double* out) {
    __shared__ double red[256];
    double s = 0.0;
    for (int64_t i = threadIdx.x; i < nblk; i += blockDim.x) s += logd[i];
    red[threadIdx.x] = s;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
        __syncthreads();
    }
    const double logdet = 2.0 * red[0];
    __syncthreads();
    for (int j = 0; j < k; ++j) {
        double q = 0.0;
        for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
            const double v = Z[(int64_t)j * n + i];
            q += v * v;
        }
        red[threadIdx.x] = q;
        __syncthreads();
        for (int o = 128; o > 0; o >>= 1) {
            if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            const double quad = red[0];
            out[3 * j + 0] = -0.5 * (double)n * log(2.0 * 3.14159265358979323846) - 0.5 * logdet - 0.5 * quad;
            out[3 * j + 1] = logdet;
            out[3 * j + 2] = quad;
        }
        __syncthreads();
    }
}

__global__ void k_matern_block(const double* a, int64_t ni, const double* b, int64_t nj, MaternParams p, double* out) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= ni * nj) return;
    const int64_t i = idx % ni, j = idx / ni;
    const double h = dist2d(a[2 * i], a[2 * i + 1], b[2 * j], b[2 * j + 1]);
    out[idx] = matern_dev(h, p);
}

bool g_attr_set = false;
void set_attrs() {
    if (g_attr_set) return;
    HM_CUDA_TRY(cudaFuncSetAttribute(k_potrf_diag, cudaFuncAttributeMaxDynamicSharedMemorySize, 1 * TSZ * 8));
    HM_CUDA_TRY(cudaFuncSetAttribute(k_trsm_panel, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * TSZ * 8));
    HM_CUDA_TRY(cudaFuncSetAttribute(k_syrk_trailing, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * TSZ * 8));
    HM_CUDA_TRY(cudaFuncSetAttribute(k_trsv_diag, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * TSZ * 8));
    HM_CUDA_TRY(cudaFuncSetAttribute(k_solve_update, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * TSZ * 8));
    g_attr_set = true;
}

}  // namespace

// Device-side dense log-likelihood.  pts_d: n x 2 (device), Z_d: n x k device
// (overwritten with v = L^{-1} Z), work_A: n*n doubles, logd: ceil(n/64),
// fail: 1 int, out_d: 3k doubles.
void dense_loglik_device(const double* pts_d, int64_t n, const MaternParams& p, double* Z_d, int k,
                         double* work_A, double* logd, int* fail, double* out_d, cudaStream_t st) {
    set_attrs();
    HM_CUDA_TRY(cudaMemsetAsync(fail, 0, sizeof(int), st));
    dim3 bt(16, 16), bg((unsigned)((n + 15) / 16), (unsigned)((n + 15) / 16));
    k_dense_matern<<<bg, bt, 0, st>>>(work_A, n, pts_d, p);
    HM_CUDA_TRY(cudaGetLastError());
    const int64_t nblk = (n + TD - 1) / TD;
    for (int64_t jb = 0; jb < nblk; ++jb) {
        const int64_t j0 = jb * TD;
        k_potrf_diag<<<1, TTHREADS, TSZ * 8, st>>>(work_A, n, j0, logd, fail);
        const int64_t rest = nblk - jb - 1;
        if (rest > 0) {
            k_trsm_panel<<<(unsigned)rest, TTHREADS, 2 * TSZ * 8, st>>>(work_A, n, j0);
            k_syrk_trailing<<<(unsigned)(rest * (rest + 1) / 2), TTHREADS, 3 * TSZ * 8, st>>>(work_A, n, j0);
        }
    }
    HM_CUDA_TRY(cudaGetLastError());
    const int ncb = (k + TD - 1) / TD;
    for (int64_t jb = 0; jb < nblk; ++jb) {
        const int64_t j0 = jb * TD;
        k_trsv_diag<<<ncb, TTHREADS, 2 * TSZ * 8, st>>>(work_A, n, Z_d, j0, k);
        const int64_t rest = nblk - jb - 1;
        if (rest > 0) {
            dim3 g((unsigned)rest, (unsigned)ncb);
            k_solve_update<<<g, TTHREADS, 3 * TSZ * 8, st>>>(work_A, n, Z_d, j0, k);
        }
    }
    k_dense_finish<<<1, 256, 0, st>>>(logd, nblk, Z_d, n, k, out_d);
    HM_CUDA_TRY(cudaGetLastError());
}

void matern_block_device(const double* a_d, int64_t ni, const double* b_d, int64_t nj, const MaternParams& p,
                         double* out_d, cudaStream_t st) {
    const int64_t tot = ni * nj;
    if (tot == 0) return;
    k_matern_block<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(a_d, ni, b_d, nj, p, out_d);
    HM_CUDA_TRY(cudaGetLastError());
}

}  // namespace hm
