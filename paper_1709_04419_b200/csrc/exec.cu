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
#include "sched.h"
#include "api_util.h"
#include "tile.cuh"
#include "trunc.cuh"
#include "vm.cuh"

namespace hm {

constexpr int EXEC_SMEM = (VM_SMEM > TR_SMEM) ? VM_SMEM : TR_SMEM;


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

// ---- ready-queue executor (sched.h) ---------------------------------------
// Tasks are claimed only once ready: a finishing task increments the arrival
// counter of each successor (acq_rel atomics) and the last arrival pushes the
// successor (a cooperative group: nsub consecutive slots) to its priority
// queue.  Warp 0 of an idle CTA reads all RQ_NQ {head, tail} pairs at once
// (one lane per queue), claims the first non-empty one in priority order by a
// CAS on its head and waits for the slot to be published.  No CTA ever spins
// on an unfinished predecessor, and a task on the critical path (high bottom
// level) overtakes ready work of lower priority.
// Deadlock freedom: a CTA blocks only in a cooperative group barrier; a group
// occupies consecutive slots of one queue and slots are claimed in order, so at
// most one group per coop queue is partially claimed: <= RQ_NCOOP * (TR_COOP_MAX
// - 1) blocked CTAs < grid (checked at launch), the rest keep claiming.
__device__ __forceinline__ long long ld_relaxed_gpu64(const long long* p) {
    long long v;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ int atom_add_acqrel_gpu(int* p, int v) {
    int old;
    asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}

__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

__device__ __forceinline__ void st_relaxed_gpu(int* p, int v) {
    asm volatile("st.relaxed.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// xr: the phase's tasks with (dep_begin, dep_count) replaced by their successor range in
// succ2 = {successor, rq_pack(need, nsub, queue)} pairs (sched.h)
// one CTA per SM: the whole register file (no spills of the truncation code) and an
// SM of its own for a critical-path task beat a second resident CTA (measured at
// n = 64k: H-Cholesky 652 -> ~560 ms)
#ifndef HM_EXEC_RQ_MINB
#define HM_EXEC_RQ_MINB 1
#endif
__global__ void __launch_bounds__(TTHREADS, HM_EXEC_RQ_MINB)
    k_exec_rq(const XTask* __restrict__ xr, int nx, const int2* __restrict__ succ2, const int32_t* __restrict__ qbase,
              int* cnt, int* slot, int* ctl, const VTask* __restrict__ vt, const VIns* __restrict__ ins,
              const VTerm* __restrict__ terms, const TTask* __restrict__ tt, const TPiece* __restrict__ tp,
              double* pool, int* ranks, int* flags, double* ctr, double eps, unsigned long long* trace, int* bars) {
    extern __shared__ double sm[];
    __shared__ int s_task;
    __shared__ int2 s_succ[32];
    const int lane = threadIdx.x & 31;
    int* finished = ctl + 2 * RQ_NQ;
    int next = -1;   // continuation: a successor this CTA made ready and kept for itself (warp 0)
    for (;;) {
        if (threadIdx.x < 32) {
            if (next >= 0) {
                // the completion fence of the previous task (below) already ordered and
                // invalidated what this one reads
                if (lane == 0) s_task = next;
            } else {
                int got = -1;
                for (;;) {
                    int h = 0, t = 0;
                    if (lane < RQ_NQ) {
                        const long long ht = ld_relaxed_gpu64(reinterpret_cast<const long long*>(ctl) + lane);
                        h = (int)(ht & 0xffffffffll);
                        t = (int)(ht >> 32);
                    }
                    const unsigned m = __ballot_sync(0xffffffffu, lane < RQ_NQ && h < t);
                    if (m) {
                        const int q = __ffs(m) - 1;
                        int ok = 0;
                        if (lane == q) ok = (atomicCAS(ctl + 2 * q, h, h + 1) == h);
                        ok = __shfl_sync(0xffffffffu, ok, q);
                        if (ok) {
                            got = qbase[q] + __shfl_sync(0xffffffffu, h, q);
                            break;
                        }
                        continue;
                    }
                    int fin = 0;
                    if (lane == 0) fin = (ld_acquire_gpu(finished) >= nx);
                    if (__shfl_sync(0xffffffffu, fin, 0)) break;
                    __nanosleep(128);
                }
                if (lane == 0) {
                    int task = -1;
                    if (got >= 0)
                        while ((task = ld_acquire_gpu(slot + got)) < 0) __nanosleep(20);
                    s_task = task;
                }
                __syncwarp();
                if (lane == 0) fence_acq_rel_gpu();
            }
        }
        __syncthreads();
        const int i = s_task;
        __syncthreads();
        if (i < 0) return;
        const XTask x = xr[i];
        unsigned long long t_claim = 0;
        if (trace && threadIdx.x == 0) t_claim = gtimer();
        // stage the first 32 successor records while the task runs
        if (threadIdx.x < 32) {
            const bool v = lane < x.dep_count;
            cp_async8(reinterpret_cast<double*>(s_succ + lane),
                      reinterpret_cast<const double*>(succ2 + x.dep_begin + (v ? lane : 0)), v);
            cp_async_commit();
        }
        unsigned long long* stt = trace ? trace + 4 * (size_t)nx + 64 * (size_t)i : nullptr;
        if (x.kind == 0) vm_run(vt[x.idx], ins, terms, pool, ranks, flags, ctr, sm, stt);
        else {
            const TTask t = tt[x.idx];
            trunc_run(t, tp, pool, ranks, flags, eps, ctr, sm, x.sub, x.nsub, bars + t.bar, stt);
        }
        if (threadIdx.x < 32) cp_async_wait<0>();
        __syncthreads();
        if (threadIdx.x < 32) {
            // release this task's writes (the CTA's, ordered before by the barrier); then count
            // the arrival at every successor (a successor with a single predecessor needs no
            // counter); the last arrival owns the successor: it keeps the most urgent ready
            // single task as its continuation and pushes the others
            fence_acq_rel_gpu();
            next = -1;
            for (int kb = 0; kb < x.dep_count; kb += 32) {
                const int k = kb + lane;
                int s = -1, pk = 0, key = 0x7fffffff;
                bool counted = false;
                if (k < x.dep_count) {
                    const int2 e = (kb == 0) ? s_succ[lane] : succ2[x.dep_begin + k];
                    pk = e.y;
                    const int need = pk >> RQ_NEED_SHIFT;
                    counted = need > 1;
                    if (!counted || atomicAdd(cnt + e.x, 1) + 1 == need) {
                        s = e.x;
                        key = (((pk >> RQ_NSUB_SHIFT) & 63) == 1) ? (pk & 31) : 0x7ffffffe;
                    }
                }
                if (__ballot_sync(0xffffffffu, s >= 0) == 0u) continue;
                // acquire the other predecessors' writes before handing such a successor on
                if (__ballot_sync(0xffffffffu, s >= 0 && counted)) fence_acq_rel_gpu();
                int best = key;
                if (next < 0) {
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) best = min(best, __shfl_xor_sync(0xffffffffu, best, o));
                }
                const unsigned win = __ballot_sync(0xffffffffu, next < 0 && s >= 0 && key == best && best < 0x7ffffffe);
                const int wl = win ? __ffs(win) - 1 : -1;
                if (wl >= 0) next = __shfl_sync(0xffffffffu, s, wl);
                if (s >= 0 && lane != wl) {
                    // the fence above makes this plain store a release of everything seen so far
                    const int ns = (pk >> RQ_NSUB_SHIFT) & 63, q = pk & 31;
                    const int pos = qbase[q] + atomicAdd(ctl + 2 * q + 1, ns);
                    for (int j = 0; j < ns; ++j) st_relaxed_gpu(slot + pos + j, s + j);
                }
            }
            __syncwarp();
            if (lane == 0) {
                atomicAdd(finished, 1);
                if (trace) {
                    const unsigned long long t_end = gtimer();
                    if (x.kind == 0) stt[5] = t_end;
                    unsigned int smid;
                    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
                    trace[4 * (size_t)i + 0] = t_claim;
                    trace[4 * (size_t)i + 1] = t_claim;
                    trace[4 * (size_t)i + 2] = t_end;
                    trace[4 * (size_t)i + 3] = smid | ((unsigned long long)x.kind << 16) | ((unsigned long long)blockIdx.x << 32);
                }
            }
        }
    }
}

static int grid_of(const void* fn, int& cache) {
    if (cache) return cache;
    HM_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, EXEC_SMEM));
    int dev = 0, sms = 0, occ = 0;
    HM_CUDA_TRY(cudaGetDevice(&dev));
    HM_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    HM_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, TTHREADS, EXEC_SMEM));
    if (occ < 1) occ = 1;
    int grid = sms * occ;
    if (const char* g = std::getenv("HM_EXEC_GRID")) {   // debug: fewer persistent CTAs
        const int v = std::atoi(g);
        if (v > 0 && v < grid) grid = v;
    }
    cache = grid;
    return grid;
}

int exec_grid() {
    static int g = 0;
    return grid_of((const void*)k_exec, g);
}

int exec_grid_rq() {
    static int g = 0;
    return grid_of((const void*)k_exec_rq, g);
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

void launch_exec_rq(const XTask* xr, int nx, const int32_t* succ2, const int32_t* qbase, const int32_t* slot_init, const int32_t* ctl_init,
                    int* cnt, int* slot, int* ctl, const VTask* vt, const VIns* ins, const VTerm* terms, const TTask* tt,
                    const TPiece* tp, double* pool, int* ranks, int* flags, double* ctr, double eps,
                    unsigned long long* trace, int* bars, int nbars, int max_nsub, int grid_cap, cudaStream_t st) {
    if (nx <= 0) return;
    int grid = exec_grid_rq();
    if (grid_cap > 0 && grid_cap < grid) grid = grid_cap;
    // deadlock freedom: CTAs blocked in partially claimed groups (<= RQ_NCOOP groups) < grid
    if (grid <= RQ_NCOOP * (max_nsub - 1)) throw ApiError(HM_ERR_ARG, "ready-queue executor needs more resident CTAs");
    HM_CUDA_TRY(cudaMemsetAsync(cnt, 0, sizeof(int) * nx, st));
    HM_CUDA_TRY(cudaMemcpyAsync(slot, slot_init, sizeof(int) * nx, cudaMemcpyDeviceToDevice, st));
    HM_CUDA_TRY(cudaMemcpyAsync(ctl, ctl_init, sizeof(int) * (2 * RQ_NQ + 2), cudaMemcpyDeviceToDevice, st));
    if (nbars > 0) HM_CUDA_TRY(cudaMemsetAsync(bars, 0, sizeof(int) * nbars, st));
    k_exec_rq<<<grid, TTHREADS, EXEC_SMEM, st>>>(xr, nx, reinterpret_cast<const int2*>(succ2), qbase, cnt, slot, ctl, vt, ins, terms, tt, tp, pool, ranks, flags, ctr, eps,
                                                 trace, bars);
}

}  // namespace hm
