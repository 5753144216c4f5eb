#pragma once
#include <cuda_runtime.h>

#include "common.h"
#include "hm_tasks.h"

namespace hm {
// Device work counters (doubles): [CTR_x + 0] algorithmic flops (or kernel
// evaluations for DGEN), [CTR_x + 1] algorithmic bytes, accumulated by the kernels.
constexpr int CTR_DGEN = 0, CTR_ACA = 2, CTR_TRUNC = 4, CTR_VM = 6, CTR_N = 8;
void launch_dense_gen(const DenseGenTask* t, int n, const double* pts, double* pool, const MaternParams& p,
                      double* ctr, cudaStream_t st);
void launch_aca(const AcaTask* t, int n, const double* pts, double* pool, int* ranks, int* flags,
                const MaternParams& p, double eps, double* ctr, cudaStream_t st);
void launch_trunc(const TTask* t, int n, const TPiece* pc, double* pool, int* ranks, int* flags, double eps,
                  double* ctr, cudaStream_t st);
void vm_set_attr();
void launch_vm(const VTask* t, int n, const VIns* ins, const VTerm* terms, double* pool, const int* ranks, int* flags,
               double* ctr, cudaStream_t st);
int exec_grid();
int exec_grid_rq();
void launch_exec(const XTask* xt, int nx, const int32_t* deps, const VTask* vt, const VIns* ins, const VTerm* terms,
                 const TTask* tt,
                 const TPiece* tp, double* pool, int* ranks, int* flags, double* ctr, double eps, int* done,
                 int* counter, int epoch, unsigned long long* trace, int* bars, int nbars, cudaStream_t st);
void launch_exec_rq(const XTask* xr, int nx, const int32_t* succ2, const int32_t* qbase, const int32_t* slot_init, const int32_t* ctl_init,
                    int* cnt, int* slot, int* ctl, const VTask* vt, const VIns* ins, const VTerm* terms, const TTask* tt,
                    const TPiece* tp, double* pool, int* ranks, int* flags, double* ctr, double eps,
                    unsigned long long* trace, int* bars, int nbars, int max_nsub, int grid_cap, cudaStream_t st);
void launch_gather(const double* Z, const int64_t* perm, int64_t n, int kz, int zw, double* Zt, cudaStream_t st);
void launch_scatter(const double* Zt, const int64_t* perm, int64_t n, int kz, double* Z, cudaStream_t st);
void launch_set_int(int* p, int v, cudaStream_t st);   // z-buffer column count -> its rank slot
void launch_finish(const double* logd, int nleaves, const double* Zt, int64_t n, int kz, double* out,
                   cudaStream_t st);
}  // namespace hm
