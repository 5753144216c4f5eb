#pragma once
#include <cuda_runtime.h>

#include "common.h"
#include "hm_tasks.h"

namespace hm {
void launch_dense_gen(const DenseGenTask* t, int n, const double* pts, double* pool, const MaternParams& p,
                      cudaStream_t st);
void launch_aca(const AcaTask* t, int n, const double* pts, double* pool, int* ranks, int* flags,
                const MaternParams& p, double eps, cudaStream_t st);
void launch_trunc(const TTask* t, int n, const TPiece* pc, double* pool, int* ranks, int* flags, double eps,
                  cudaStream_t st);
void vm_set_attr();
void launch_vm(const VTask* t, int n, const VIns* ins, double* pool, const int* ranks, int* flags, cudaStream_t st);
void launch_gather(const double* Z, const int64_t* perm, int64_t n, int kz, int zw, double* Zt, cudaStream_t st);
void launch_scatter(const double* Zt, const int64_t* perm, int64_t n, int kz, double* Z, cudaStream_t st);
void launch_finish(const double* logd, int nleaves, const double* Zt, int64_t n, int kz, double* out,
                   cudaStream_t st);
}  // namespace hm
