// Tile VM: one CTA executes a short program (hm_tasks.h VmOp) on NTILE 64 x 64
// fp64 shared-memory tiles -- leaf-level POTRF / TRSM / TRMM and the products of
// the H-Cholesky, solves and sampler (sec. 3.1, l.259-283).
#pragma once
#include <cuda_runtime.h>

#include "dev_util.cuh"
#include "hm_kernels.h"
#include "hm_tasks.h"
#include "tile.cuh"

namespace hm {

// Execute one tile-VM program with the CTA (TTHREADS threads); sm = NTILE tiles.
__device__ __forceinline__ void vm_run(const VTask task, const VIns* __restrict__ ins, double* pool, const int* ranks,
                                       int* flags, double* ctr, double* sm) {
    __shared__ int trows[NTILE], tcols[NTILE];
    __shared__ double s_log;
    double c_fl = 0.0, c_by = 0.0;   // algorithmic flops / bytes of this program (thread 0)
    for (int pc = 0; pc < task.ins_count; ++pc) {
        const VIns I = ins[task.ins_begin + pc];
        double* T0 = sm + (int)I.t0 * TSZ;
        switch (I.op) {
            case VM_LD: {
                const int r = dim_eval(I.rows, ranks), c = dim_eval(I.cols, ranks);
                tile_load(T0, pool + I.goff, I.ld, r, c);
                if (threadIdx.x == 0) { trows[I.t0] = r; tcols[I.t0] = c; c_by += 8.0 * r * c; }
                __syncthreads();
            } break;
            case VM_ST: {
                const int r = dim_eval(I.rows, ranks), c = dim_eval(I.cols, ranks);
                tile_store(T0, pool + I.goff, I.ld, min(r, trows[I.t0]), min(c, tcols[I.t0]));
                if (threadIdx.x == 0) c_by += 8.0 * min(r, trows[I.t0]) * min(c, tcols[I.t0]);
                __syncthreads();
            } break;
            case VM_ZERO: {
                tile_zero(T0);
                if (threadIdx.x == 0) {
                    trows[I.t0] = dim_eval(I.rows, ranks);
                    tcols[I.t0] = dim_eval(I.cols, ranks);
                }
                __syncthreads();
            } break;
            case VM_GEMM: {
                const double* T1 = sm + (int)I.t1 * TSZ;
                const double* T2 = sm + (int)I.t2 * TSZ;
                const int m = I.ta ? tcols[I.t1] : trows[I.t1];
                const int ka = I.ta ? trows[I.t1] : tcols[I.t1];
                const int kb = I.tb ? tcols[I.t2] : trows[I.t2];
                const int n = I.tb ? trows[I.t2] : tcols[I.t2];
                const int k = max(ka, kb);
                if (I.beta == 0.0) {
                    tile_zero(T0);
                    __syncthreads();
                    if (threadIdx.x == 0) { trows[I.t0] = m; tcols[I.t0] = n; }
                }
                if (threadIdx.x == 0) c_fl += 2.0 * m * n * k;
                if (m > 0 && n > 0 && k > 0)
                    tile_gemm(T0, T1, I.ta != 0, T2, I.tb != 0, m, n, k, I.alpha, I.beta == 0.0 ? 0.0 : I.beta);
                __syncthreads();
            } break;
            case VM_POTRF: {
                if (threadIdx.x == 0) c_fl += (double)trows[I.t0] * trows[I.t0] * trows[I.t0] / 3.0;
                const int f = tile_potrf(T0, trows[I.t0], &s_log);
                if (threadIdx.x == 0) {
                    pool[I.goff] = s_log;
                    if (f) atomicAdd(flags, f);
                }
                __syncthreads();
            } break;
            case VM_TRSM_RLT: {
                if (threadIdx.x == 0) c_fl += (double)trows[I.t0] * tcols[I.t0] * tcols[I.t0];
                tile_trsm_rlt(T0, sm + (int)I.t1 * TSZ, trows[I.t0], tcols[I.t0]);
            } break;
            case VM_TRSM_LN: {
                if (threadIdx.x == 0) c_fl += (double)trows[I.t0] * trows[I.t0] * tcols[I.t0];
                tile_trsm_ln(T0, sm + (int)I.t1 * TSZ, trows[I.t0], tcols[I.t0]);
            } break;
            case VM_TRMM_LN: {
                if (threadIdx.x == 0) c_fl += (double)trows[I.t0] * trows[I.t0] * tcols[I.t0];
                tile_trmm_ln(T0, sm + (int)I.t1 * TSZ, trows[I.t0], tcols[I.t0]);
            } break;
            default:
                break;
        }
    }
    if (threadIdx.x == 0) {
        atomicAdd(ctr + CTR_VM + 0, c_fl);
        atomicAdd(ctr + CTR_VM + 1, c_by);
    }
}

}  // namespace hm
