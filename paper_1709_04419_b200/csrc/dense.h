#pragma once
#include <cuda_runtime.h>

#include "common.h"

namespace hm {

void dense_loglik_device(const double* pts_d, int64_t n, const MaternParams& p, double* Z_d, int k,
                         double* work_A, double* logd, int* fail, double* out_d, cudaStream_t st);

void matern_block_device(const double* a_d, int64_t ni, const double* b_d, int64_t nj, const MaternParams& p,
                         double* out_d, cudaStream_t st);

}  // namespace hm
