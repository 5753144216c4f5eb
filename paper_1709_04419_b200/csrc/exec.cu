// Persistent dependency-driven executor of a planned phase (H-Cholesky, solve,
// sampler, recompression): one CTA per SM claims tasks in the planner's
// topological order (global atomic counter), waits until every predecessor has
// published completion (done[p] == epoch, acquire), runs the task -- a tile-VM
// program (vm.cuh) or a low-rank truncation (trunc.cuh) -- and publishes its own
// completion (release).  Claiming in topological order with all CTAs resident
// makes the wait deadlock-free: the lowest unfinished claimed task always has
// all its predecessors finished.  This replaces one launch (and one grid-wide
// barrier) per wave by fine-grained edges, so independent tasks of different
// waves overlap.
#include <cuda_runtime.h>

#include <cstdlib>

#include "dev_util.cuh"
#include "hm_kernels.h"
#include "hm_tasks.h"
#include "tile.cuh"
#include "trunc.cuh"
#include "vm.cuh"

namespace hm {

constexpr int EXEC_SMEM = (NTILE * TSZ * 8 > TR_SMEM) ? NTILE * TSZ * 8 : TR_SMEM;


__global__ void __launch_bounds__(TTHREADS, 2)
    k_exec(const XTask* __restrict__ xt, int nx, const int32_t* __restrict__ deps, const VTask* __restrict__ vt,
           const VIns* __restrict__ ins, const VTerm* __restrict__ terms, const TTask* __restrict__ tt, const TPiece* __restrict__ tp, double* pool,
           int* ranks, int* flags, double* ctr, double eps, int* done, int* counter, int epoch,
           unsigned long long* trace, int* bars) {
    extern __shared__ double sm[];
    __shared__ int s_task;
    for (;;) {
        if (threadIdx.x == 0) s_task = atomicAdd(counter, 1);
        __syncthreads();
        const int i = s_task;
        __syncthreads();
        if (i >= nx) return;
        const XTask x = xt[i];
        unsigned long long t_claim = 0, t_ready = 0;
        if (trace && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_claim));
        if (threadIdx.x < 32) {
            for (int d = threadIdx.x; d < x.dep_count; d += 32) {
                const int* f = done + deps[x.dep_begin + d];
                while (ld_acquire_gpu(f) != epoch) __nanosleep(40);
            }
            __syncwarp();
            if (threadIdx.x == 0) asm volatile("fence.acq_rel.gpu;" ::: "memory");
        }
        __syncthreads();
        if (trace && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_ready));
        if (x.kind == 0) vm_run(vt[x.idx], ins, terms, pool, ranks, flags, ctr, sm);
        else {
            const TTask t = tt[x.idx];
            trunc_run(t, tp, pool, ranks, flags, eps, ctr, sm, x.sub, x.nsub, bars + t.bar,
                      trace ? trace + 4 * (size_t)nx + 64 * (size_t)i : nullptr);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            st_release_gpu(done + i, epoch);
            if (trace) {   // per task: claim, ready (deps satisfied), end [ns], sm id | kind << 16
                unsigned long long t_end;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
                unsigned int smid;
                asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
                trace[4 * (size_t)i + 0] = t_claim;
                trace[4 * (size_t)i + 1] = t_ready;
                trace[4 * (size_t)i + 2] = t_end;
                trace[4 * (size_t)i + 3] = smid | ((unsigned long long)x.kind << 16) | ((unsigned long long)blockIdx.x << 32);
            }
        }
    }
}

int exec_grid() {
    static int grid = 0;
    if (grid) return grid;
    HM_CUDA_TRY(cudaFuncSetAttribute(k_exec, cudaFuncAttributeMaxDynamicSharedMemorySize, EXEC_SMEM));
    int dev = 0, sms = 0, occ = 0;
    HM_CUDA_TRY(cudaGetDevice(&dev));
    HM_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    HM_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_exec, TTHREADS, EXEC_SMEM));
    if (occ < 1) occ = 1;
    grid = sms * occ;
    if (const char* g = std::getenv("HM_EXEC_GRID")) {   // debug: fewer persistent CTAs
        const int v = std::atoi(g);
        if (v > 0 && v < grid) grid = v;
    }
    return grid;
}

void launch_exec(const XTask* xt, int nx, const int32_t* deps, const VTask* vt, const VIns* ins, const VTerm* terms,
                 const TTask* tt,
                 const TPiece* tp, double* pool, int* ranks, int* flags, double* ctr, double eps, int* done,
                 int* counter, int epoch, unsigned long long* trace, int* bars, int nbars, cudaStream_t st) {
    if (nx <= 0) return;
    const int grid = exec_grid();
    HM_CUDA_TRY(cudaMemsetAsync(counter, 0, sizeof(int), st));
    if (nbars > 0) HM_CUDA_TRY(cudaMemsetAsync(bars, 0, sizeof(int) * nbars, st));
    k_exec<<<grid, TTHREADS, EXEC_SMEM, st>>>(xt, nx, deps, vt, ins, terms, tt, tp, pool, ranks, flags, ctr, eps, done,
                                              counter, epoch, trace, bars);
}

}  // namespace hm
