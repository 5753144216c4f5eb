// k_trunc: one CTA per truncation task (algorithms in trunc.cuh).
#include "trunc.cuh"

namespace hm {

__global__ void __launch_bounds__(TR_THREADS) k_trunc(const TTask* __restrict__ tasks, const TPiece* __restrict__ pieces,
                                                      double* __restrict__ pool, int* __restrict__ ranks,
                                                      int* __restrict__ flags, double eps, double* __restrict__ ctr) {
    trunc_run(tasks[blockIdx.x], pieces, pool, ranks, flags, eps, ctr);
}

void launch_trunc(const TTask* t, int n, const TPiece* pc, double* pool, int* ranks, int* flags, double eps,
                  double* ctr, cudaStream_t st) {
    if (n > 0) k_trunc<<<n, TR_THREADS, 0, st>>>(t, pc, pool, ranks, flags, eps, ctr);
}

}  // namespace hm
