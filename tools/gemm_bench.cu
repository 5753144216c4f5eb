// Microbenchmark of the CTA-level DMMA GEMM (paper_1709_04419_b200/csrc/gemm.cuh):
// one CTA (the truncation's situation) and a full grid, per shape; checks the
// result against a simple reference kernel.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include "../paper_1709_04419_b200/csrc/gemm.cuh"
using namespace hm;

template <int SHAPE, bool TA, bool TB>
__device__ void gemm_shape(int M, int N, int K, const double* A, int lda, const double* B, int ldb, double* C, int ldc,
                           double* sm) {
    if (SHAPE == 0) gemm_wide<TA, TB>(M, N, K, 1.0, gop(A, lda, TA), gop(B, ldb, TB), 0.0, C, ldc, blockIdx.x, gridDim.x, sm);
    if (SHAPE == 1) gemm_narrow<TA, TB>(M, N, K, 1.0, gop(A, lda, TA), gop(B, ldb, TB), 0.0, C, ldc, blockIdx.x, gridDim.x, sm);
    if (SHAPE == 2) gemm_short<TA, TB>(M, N, K, 1.0, gop(A, lda, TA), gop(B, ldb, TB), 0.0, C, ldc, blockIdx.x, gridDim.x, sm);
}
template <int SHAPE>
__global__ void kgemm(int M, int N, int K, const double* A, int lda, bool tA, const double* B, int ldb, bool tB,
                      double* C, int ldc, int reps) {
    extern __shared__ double sm[];
    for (int r = 0; r < reps; ++r) {
        if (tA && tB) gemm_shape<SHAPE, true, true>(M, N, K, A, lda, B, ldb, C, ldc, sm);
        if (tA && !tB) gemm_shape<SHAPE, true, false>(M, N, K, A, lda, B, ldb, C, ldc, sm);
        if (!tA && tB) gemm_shape<SHAPE, false, true>(M, N, K, A, lda, B, ldb, C, ldc, sm);
        if (!tA && !tB) gemm_shape<SHAPE, false, false>(M, N, K, A, lda, B, ldb, C, ldc, sm);
    }
}
__global__ void kref(int M, int N, int K, const double* A, int lda, bool tA, const double* B, int ldb, bool tB, double* C,
                     int ldc) {
    int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y;
    if (i >= M || j >= N) return;
    double s = 0;
    for (int k = 0; k < K; ++k) s += (tA ? A[k + (size_t)i * lda] : A[i + (size_t)k * lda]) * (tB ? B[j + (size_t)k * ldb] : B[k + (size_t)j * ldb]);
    C[i + (size_t)j * ldc] = s;
}
template <int SHAPE>
void run(const char* name, int M, int N, int K, bool tA, bool tB, int grid) {
    int lda = tA ? K : M, ldb = tB ? N : K;
    size_t na = (size_t)lda * (tA ? M : K), nb = (size_t)ldb * (tB ? K : N);
    std::vector<double> ha(na), hb(nb);
    for (auto& x : ha) x = rand() / (double)RAND_MAX - 0.5;
    for (auto& x : hb) x = rand() / (double)RAND_MAX - 0.5;
    double *A, *B, *C, *R;
    cudaMalloc(&A, na * 8); cudaMalloc(&B, nb * 8); cudaMalloc(&C, (size_t)M * N * 8); cudaMalloc(&R, (size_t)M * N * 8);
    cudaMemcpy(A, ha.data(), na * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(B, hb.data(), nb * 8, cudaMemcpyHostToDevice);
    const int smem = GEMM_SMEM_DOUBLES * 8;
    cudaFuncSetAttribute(kgemm<SHAPE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    kgemm<SHAPE><<<grid, 256, smem>>>(M, N, K, A, lda, tA, B, ldb, tB, C, M, 1);
    kref<<<dim3((M + 127) / 128, N), 128>>>(M, N, K, A, lda, tA, B, ldb, tB, R, M);
    std::vector<double> hc((size_t)M * N), hr((size_t)M * N);
    cudaMemcpy(hc.data(), C, hc.size() * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(hr.data(), R, hr.size() * 8, cudaMemcpyDeviceToHost);
    double err = 0, mx = 0;
    for (size_t i = 0; i < hc.size(); ++i) { err = fmax(err, fabs(hc[i] - hr[i])); mx = fmax(mx, fabs(hr[i])); }
    const int reps = 20;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    kgemm<SHAPE><<<grid, 256, smem>>>(M, N, K, A, lda, tA, B, ldb, tB, C, M, reps);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double us = ms * 1e3 / reps;
    printf("%-8s M=%5d N=%5d K=%5d tA=%d tB=%d grid=%3d: %9.1f us  %8.1f GF/s  relerr=%.1e %s\n", name, M, N, K, tA, tB,
           grid, us, 2.0 * M * N * K / us / 1e3, err / mx, cudaGetErrorString(cudaGetLastError()));
    cudaFree(A); cudaFree(B); cudaFree(C); cudaFree(R);
}
int main() {
    run<1>("narrow", 256, 16, 1700, false, true, 1);      // R3: Y = Ast T
    run<2>("short", 16, 1500, 128, true, false, 1);       // R2 small
    run<2>("short", 16, 1700, 256, true, false, 1);       // R2: T^T = Om^T Bst
    run<0>("wide", 48, 1700, 256, true, false, 1);        // F1: P^T = Q^T Ast
    run<0>("wide", 256, 48, 1700, false, true, 1);        // F2: W = Bst P
    run<2>("short", 112, 16, 4096, true, false, 1);       // proj: C = Q^T Y
    run<0>("wide", 4096, 64, 1700, false, true, 26);      // big F2 on a group
    // ragged / odd leading dimensions (8-byte fallback copies, half-valid pairs)
    run<0>("wide", 255, 37, 301, false, false, 4);
    run<0>("wide", 255, 37, 301, true, true, 4);
    run<1>("narrow", 130, 16, 257, true, false, 2);
    run<2>("short", 16, 131, 255, false, true, 2);
    run<1>("narrow", 80, 16, 64, true, false, 1);         // proj: Q^T Y on one row chunk
    run<0>("wide", 8192, 8192, 64, false, true, 148);     // throughput check
    run<0>("wide", 2048, 2048, 2048, false, false, 148);
    return 0;
}
