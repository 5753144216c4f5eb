// Small device helpers shared by the H-matrix kernels (header-only, inlined).
#pragma once
#include <cuda_runtime.h>

#include "hm_tasks.h"

namespace hm {

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_gpu(int* p, int v) {
    asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// ranks are produced by other CTAs of the persistent executor: read through L2 (ld.cg)
__device__ __forceinline__ int dim_eval(const Dim& d, const int* ranks) {
    if (d.slot < 0) return d.stat;
    int v = __ldcg(ranks + d.slot) - d.off;
    return v < 0 ? 0 : (v > d.stat ? d.stat : v);
}

// ---------------------------------------------------------------- reductions
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// block-wide sum (all threads get the result); scratch >= 32 doubles
__device__ __forceinline__ double block_sum(double v, double* scratch) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) scratch[warp] = v;
    __syncthreads();
    double s = 0.0;
    for (int i = 0; i < nw; ++i) s += scratch[i];
    __syncthreads();
    return s;
}

// block-wide argmax of |v| (ties -> smaller index); returns index, *best = value
__device__ __forceinline__ int block_argmax(double v, int idx, double* best, double* sv, int* si) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    double a = fabs(v);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        double a2 = __shfl_xor_sync(0xffffffffu, a, o);
        int i2 = __shfl_xor_sync(0xffffffffu, idx, o);
        if (a2 > a || (a2 == a && i2 < idx)) { a = a2; idx = i2; }
    }
    __syncthreads();
    if (lane == 0) { sv[warp] = a; si[warp] = idx; }
    __syncthreads();
    double ba = -1.0;
    int bi = 0x7fffffff;
    for (int i = 0; i < nw; ++i)
        if (sv[i] > ba || (sv[i] == ba && si[i] < bi)) { ba = sv[i]; bi = si[i]; }
    __syncthreads();
    *best = ba;
    return bi;
}

}  // namespace hm
