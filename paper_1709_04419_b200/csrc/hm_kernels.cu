// Device kernels of the H-matrix path (sec. 2-3):
//   k_dense_gen  -- Matern entries of dense (inadmissible / leaf-pair) blocks      Eq. (2)
//   k_aca        -- partially pivoted ACA of admissible blocks to accuracy eps      l.147
//   (k_trunc, the low-rank truncation, lives in trunc.cu)
//   k_vm         -- tile VM: leaf-level POTRF / TRSM / products on 64 x 64 fp64
//                   shared-memory tiles with FP64 tensor-core MMA (see tile.cuh)
//   k_gather / k_scatter / k_finish -- permutation to tree order, log det
//                   = 2 sum log L_ii (l.283) and quad = v^T v (l.265).
#include <cuda_runtime.h>

#include <cfloat>
#include <cmath>

#include "common.h"
#include "hm_kernels.h"
#include "hm_tasks.h"
#include "matern.cuh"
#include "tile.cuh"
#include "dev_util.cuh"
#include "vm.cuh"

namespace hm {

// ---------------------------------------------------------------- assembly
__global__ void k_dense_gen(const DenseGenTask* __restrict__ tasks, const double* __restrict__ pts,
                            double* __restrict__ pool, const MaternParams p, double* __restrict__ ctr) {
    const DenseGenTask t = tasks[blockIdx.x];
    if (threadIdx.x == 0) {   // algorithmic work: m q kernel evaluations, m q doubles written
        atomicAdd(ctr + CTR_DGEN + 0, (double)t.m * t.q);
        atomicAdd(ctr + CTR_DGEN + 1, 8.0 * t.m * t.q);
    }
    double* D = pool + t.off;
    const int tot = t.m * t.q;
    for (int idx = threadIdx.x; idx < tot; idx += blockDim.x) {
        const int i = idx % t.m, j = idx / t.m;
        const int64_t gi = t.r0 + i, gj = t.c0 + j;
        const double h = dist2d(pts[2 * gi], pts[2 * gi + 1], pts[2 * gj], pts[2 * gj + 1]);
        D[idx] = (gi == gj) ? p.sigma2 : matern_dev(h, p);
    }
}

constexpr int ACA_THREADS = 256;
constexpr int ACA_MAXK = 1024;

// Adaptive cross approximation with partial pivoting (Bebendorf): pivot row i*
// -> residual row, pivot column j* = argmax |row| -> residual column; stop when
// ||u_k|| ||v_k|| <= eps ||S_k||_F, ||S_k||_F^2 updated incrementally.
__global__ void __launch_bounds__(ACA_THREADS) k_aca(const AcaTask* __restrict__ tasks, const double* __restrict__ pts,
                                                     double* __restrict__ pool, int* __restrict__ ranks,
                                                     int* __restrict__ flags, const MaternParams p, double eps,
                                                     double* __restrict__ ctr) {
    const AcaTask t = tasks[blockIdx.x];
    double* U = pool + t.u_off;
    double* V = pool + t.v_off;
    const int m = t.m, q = t.q, cap = t.cap;
    __shared__ double coef[ACA_MAXK];
    __shared__ double dots[ACA_MAXK];
    __shared__ int used[ACA_MAXK + 8];
    __shared__ double sv[32];
    __shared__ int si[32];
    __shared__ double scratch[32];
    int nused = 0;
    int istar = 0;
    int k = 0;
    double normS2 = 0.0;
    int tries = 0;
    while (k < cap) {
        // ---- residual row istar -> V[:, k]
        const double xi = pts[2 * (t.r0 + istar)], yi = pts[2 * (t.r0 + istar) + 1];
        for (int l = threadIdx.x; l < k; l += blockDim.x) coef[l] = U[istar + (int64_t)l * m];
        __syncthreads();
        double bv = 0.0;
        int bj = 0x7fffffff;
        for (int j = threadIdx.x; j < q; j += blockDim.x) {
            const int64_t gj = t.c0 + j;
            double v = matern_dev(dist2d(xi, yi, pts[2 * gj], pts[2 * gj + 1]), p);
            for (int l = 0; l < k; ++l) v -= coef[l] * V[j + (int64_t)l * q];
            V[j + (int64_t)k * q] = v;
            if (fabs(v) > fabs(bv) || (fabs(v) == fabs(bv) && j < bj)) { bv = v; bj = j; }
        }
        double vmax;
        const int jstar = block_argmax(bv, bj, &vmax, sv, si);
        if (threadIdx.x == 0 && nused < ACA_MAXK) used[nused] = istar;
        ++nused;
        __syncthreads();
        if (!(vmax > 0.0) || (k > 0 && vmax <= 1e-15 * sqrt(normS2 / ((double)m * q) + 1e-300))) {
            // numerically zero residual row: try another unused row, else stop
            if (++tries > 3 || nused >= m || nused >= ACA_MAXK) break;
            int cand = 0;
            for (;;) {
                bool u = false;
                for (int a = 0; a < nused; ++a) u |= (used[a] == cand);
                if (!u) break;
                ++cand;
            }
            istar = cand;
            continue;
        }
        const double delta = V[jstar + (int64_t)k * q];
        __syncthreads();   // every thread has read the pivot before its owner rescales it in place
        for (int j = threadIdx.x; j < q; j += blockDim.x) V[j + (int64_t)k * q] /= delta;
        __syncthreads();
        // ---- residual column jstar -> U[:, k]
        const double xj = pts[2 * (t.c0 + jstar)], yj = pts[2 * (t.c0 + jstar) + 1];
        for (int l = threadIdx.x; l < k; l += blockDim.x) coef[l] = V[jstar + (int64_t)l * q];
        __syncthreads();
        for (int i = threadIdx.x; i < m; i += blockDim.x) {
            const int64_t gi = t.r0 + i;
            double u = matern_dev(dist2d(pts[2 * gi], pts[2 * gi + 1], xj, yj), p);
            for (int l = 0; l < k; ++l) u -= coef[l] * U[i + (int64_t)l * m];
            U[i + (int64_t)k * m] = u;
        }
        __syncthreads();
        // ---- norms
        double a2 = 0.0, b2 = 0.0;
        for (int i = threadIdx.x; i < m; i += blockDim.x) { const double u = U[i + (int64_t)k * m]; a2 += u * u; }
        for (int j = threadIdx.x; j < q; j += blockDim.x) { const double v = V[j + (int64_t)k * q]; b2 += v * v; }
        const double nu2 = block_sum(a2, scratch);
        const double nv2 = block_sum(b2, scratch);
        // cross terms sum_{l<k} (u_k . u_l)(v_k . v_l): one warp per l
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
        for (int l = warp; l < k; l += nw) {
            double du = 0.0, dv = 0.0;
            for (int i = lane; i < m; i += 32) du += U[i + (int64_t)k * m] * U[i + (int64_t)l * m];
            for (int j = lane; j < q; j += 32) dv += V[j + (int64_t)k * q] * V[j + (int64_t)l * q];
            du = warp_sum(du);
            dv = warp_sum(dv);
            if (lane == 0) dots[l] = du * dv;
        }
        __syncthreads();
        double cross = 0.0;
        for (int l = 0; l < k; ++l) cross += dots[l];
        normS2 += 2.0 * cross + nu2 * nv2;
        ++k;
        tries = 0;
        // eps > 0: relative to ||S_k||_F;  eps < 0: absolute |eps| (hm_params.abs_eps)
        if (sqrt(nu2 * nv2) <= (eps > 0.0 ? eps * sqrt(fabs(normS2)) : -eps)) break;
        // ---- next pivot row: argmax |u_k| over unused rows
        double bu = 0.0;
        int bi = 0x7fffffff;
        for (int i = threadIdx.x; i < m; i += blockDim.x) {
            const double u = U[i + (int64_t)(k - 1) * m];
            if (fabs(u) > fabs(bu) || (fabs(u) == fabs(bu) && i < bi)) {
                bool isused = false;
                for (int a = 0; a < nused; ++a) isused |= (used[a] == i);
                if (!isused) { bu = u; bi = i; }
            }
        }
        double umax;
        int inext = block_argmax(bu, bi, &umax, sv, si);
        if (inext == 0x7fffffff || nused >= ACA_MAXK) break;
        istar = inext;
        if (k == cap && threadIdx.x == 0) atomicOr(flags + 1, 1);
    }
    if (threadIdx.x == 0) {
        ranks[t.rslot] = k;
        // algorithmic work of k ACA steps: (m + q) kernel evaluations per step plus the
        // residual updates sum_l 2 l (m + q); bytes: the k (m + q) factor entries written
        const double kk = (double)k;
        atomicAdd(ctr + CTR_ACA + 0, kk * (m + q) + kk * (kk - 1.0) * (m + q));
        atomicAdd(ctr + CTR_ACA + 1, 8.0 * kk * (m + q));
    }
}

// ---------------------------------------------------------------- tile VM
__global__ void __launch_bounds__(TTHREADS) k_vm(const VTask* __restrict__ tasks, const VIns* __restrict__ ins,
                                                 const VTerm* __restrict__ terms, double* __restrict__ pool,
                                                 const int* __restrict__ ranks, int* __restrict__ flags,
                                                 double* __restrict__ ctr) {
    extern __shared__ double sm[];
    vm_run(tasks[blockIdx.x], ins, terms, pool, ranks, flags, ctr, sm);
}

// ---------------------------------------------------------------- permutation / finish
// Zt[k + c n] = Z[perm[k] + c n] for c < kz, 0 for kz <= c < zw
__global__ void k_gather(const double* __restrict__ Z, const int64_t* __restrict__ perm, int64_t n, int kz, int zw,
                         double* __restrict__ Zt) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= n * zw) return;
    const int64_t k = idx % n, c = idx / n;
    Zt[idx] = (c < kz) ? Z[perm[k] + c * n] : 0.0;
}

__global__ void k_scatter(const double* __restrict__ Zt, const int64_t* __restrict__ perm, int64_t n, int kz,
                          double* __restrict__ Z) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= n * kz) return;
    const int64_t k = idx % n, c = idx / n;
    Z[perm[k] + c * n] = Zt[idx];
}

// out[3c + 0..2] = (loglik, logdet, quad) for columns c < kz of the solved z buffer
__global__ void k_finish(const double* __restrict__ logd, int nleaves, const double* __restrict__ Zt, int64_t n,
                         int kz, double* __restrict__ out) {
    __shared__ double scratch[32];
    double s = 0.0;
    for (int i = threadIdx.x; i < nleaves; i += blockDim.x) s += logd[i];
    const double logdet = 2.0 * block_sum(s, scratch);
    for (int c = 0; c < kz; ++c) {
        double qd = 0.0;
        for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
            const double v = Zt[i + c * n];
            qd += v * v;
        }
        const double quad = block_sum(qd, scratch);
        if (threadIdx.x == 0) {
            out[3 * c + 0] = -0.5 * (double)n * log(2.0 * 3.14159265358979323846) - 0.5 * logdet - 0.5 * quad;
            out[3 * c + 1] = logdet;
            out[3 * c + 2] = quad;
        }
    }
}

// ---------------------------------------------------------------- host launchers
void launch_dense_gen(const DenseGenTask* t, int n, const double* pts, double* pool, const MaternParams& p,
                      double* ctr, cudaStream_t st) {
    if (n > 0) k_dense_gen<<<n, 256, 0, st>>>(t, pts, pool, p, ctr);
}
void launch_aca(const AcaTask* t, int n, const double* pts, double* pool, int* ranks, int* flags,
                const MaternParams& p, double eps, double* ctr, cudaStream_t st) {
    if (n > 0) k_aca<<<n, ACA_THREADS, 0, st>>>(t, pts, pool, ranks, flags, p, eps, ctr);
}
void vm_set_attr() {
    static bool done = false;
    if (done) return;
    HM_CUDA_TRY(cudaFuncSetAttribute(k_vm, cudaFuncAttributeMaxDynamicSharedMemorySize, VM_SMEM));
    done = true;
}
void launch_vm(const VTask* t, int n, const VIns* ins, const VTerm* terms, double* pool, const int* ranks, int* flags,
               double* ctr, cudaStream_t st) {
    if (n > 0) k_vm<<<n, TTHREADS, VM_SMEM, st>>>(t, ins, terms, pool, ranks, flags, ctr);
}
void launch_gather(const double* Z, const int64_t* perm, int64_t n, int kz, int zw, double* Zt, cudaStream_t st) {
    const int64_t tot = n * zw;
    k_gather<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(Z, perm, n, kz, zw, Zt);
}
void launch_scatter(const double* Zt, const int64_t* perm, int64_t n, int kz, double* Z, cudaStream_t st) {
    const int64_t tot = n * kz;
    k_scatter<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(Zt, perm, n, kz, Z);
}
__global__ void k_set_int(int* p, int v) { *p = v; }
void launch_set_int(int* p, int v, cudaStream_t st) { k_set_int<<<1, 1, 0, st>>>(p, v); }

void launch_finish(const double* logd, int nleaves, const double* Zt, int64_t n, int kz, double* out,
                   cudaStream_t st) {
    k_finish<<<1, 512, 0, st>>>(logd, nleaves, Zt, n, kz, out);
}

}  // namespace hm
