// k_trunc: one CTA per truncation task (algorithms in trunc.cuh).
#include "trunc.cuh"

namespace hm {

__global__ void __launch_bounds__(TR_THREADS) k_trunc(const TTask* __restrict__ tasks, const TPiece* __restrict__ pieces,
                                                      double* __restrict__ pool, int* __restrict__ ranks,
                                                      int* __restrict__ flags, double eps, double* __restrict__ ctr) {
    extern __shared__ double dsm[];
    trunc_run(tasks[blockIdx.x], pieces, pool, ranks, flags, eps, ctr, dsm);
}

void launch_trunc(const TTask* t, int n, const TPiece* pc, double* pool, int* ranks, int* flags, double eps,
                  double* ctr, cudaStream_t st) {
    static bool attr = false;
    if (!attr) {
        HM_CUDA_TRY(cudaFuncSetAttribute(k_trunc, cudaFuncAttributeMaxDynamicSharedMemorySize, TR_SMEM));
        attr = true;
    }
    if (n > 0) k_trunc<<<n, TR_THREADS, TR_SMEM, st>>>(t, pc, pool, ranks, flags, eps, ctr);
}

}  // namespace hm
