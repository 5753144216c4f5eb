// Microbenchmark: FP64 peak on this GPU via DMMA (mma.sync m8n8k4 f64) and via
// DFMA, timed with CUDA events.  Used for the roofline denominator of the
// fp64 kernels (MEASURED_PEAKS.json has no fp64 entry).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dmma_loop(double* out, int iters) {
    double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
    double c[8][2];
    for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
    double s = 0;
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
    if (s == 12345.0) out[0] = s;
}
__global__ void dfma_loop(double* out, int iters) {
    double x[8];
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
    const double a = 0.999999, b = 1e-7;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
    }
    double s = 0;
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 12345.0) out[0] = s;
}
int main() {
    double* d; cudaMalloc(&d, 8);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int iters = 20000;
    for (int warps = 4; warps <= 16; warps *= 2) {
        int blocks = sms * 4;
        dmma_loop<<<blocks, 32 * warps>>>(d, 100);
        cudaEventRecord(e0);
        dmma_loop<<<blocks, 32 * warps>>>(d, iters);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double flops = 2.0 * 256 * 8 * (double)iters * blocks * warps;
        printf("DMMA warps/blk=%d blocks=%d: %.2f TFLOP/s\n", warps, blocks, flops / ms / 1e9);
        dfma_loop<<<blocks, 32 * warps>>>(d, 100);
        cudaEventRecord(e0);
        dfma_loop<<<blocks, 32 * warps>>>(d, iters);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        flops = 2.0 * 8 * (double)iters * blocks * warps * 32;
        printf("DFMA warps/blk=%d blocks=%d: %.2f TFLOP/s\n", warps, blocks, flops / ms / 1e9);
    }
    printf("SMs=%d\n", sms);
    return 0;
}
