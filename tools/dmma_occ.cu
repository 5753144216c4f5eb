// Microbenchmark: DMMA (mma.sync m8n8k4 f64) throughput per SM as a function of
// resident warps and independent accumulator chains per warp, with and without
// shared-memory operand loads (the executor runs one 8-warp CTA per SM).
#include <cstdio>
#include <cuda_runtime.h>
template <int NACC, bool LDS>
__global__ void dmma_chain(double* out, int iters) {
    __shared__ double sm[2048];
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) sm[i] = 1e-3 * i;
    __syncthreads();
    double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
    double c[NACC][2];
#pragma unroll
    for (int i = 0; i < NACC; ++i) c[i][0] = c[i][1] = 0;
    const int lane = threadIdx.x & 31;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < NACC; ++i) {
            if (LDS && (i & 1) == 0) { a = sm[(lane + 32 * i + it) & 2047]; b = sm[(lane * 3 + i + it) & 2047]; }
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
        }
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
    if (s == 12345.0) out[0] = s;
}
template <int NACC, bool LDS>
void run(int warps, int bps, int sms, double* d) {
    const int iters = 4000, blocks = sms * bps;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    dmma_chain<NACC, LDS><<<blocks, 32 * warps>>>(d, 10);
    cudaEventRecord(e0);
    dmma_chain<NACC, LDS><<<blocks, 32 * warps>>>(d, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 512.0 * NACC * (double)iters * blocks * warps;
    printf("acc/warp=%2d lds=%d warps/SM=%2d: %6.2f TFLOP/s (%5.1f GF/s per SM)\n", NACC, LDS, warps * bps,
           flops / ms / 1e9, flops / ms / 1e6 / sms);
}
int main() {
    double* d; cudaMalloc(&d, 8);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int w : {4, 8, 16, 32}) {
        run<1, false>(w, 1, sms, d); run<2, false>(w, 1, sms, d); run<4, false>(w, 1, sms, d);
        run<8, false>(w, 1, sms, d); run<16, false>(w, 1, sms, d);
        run<4, true>(w, 1, sms, d); run<8, true>(w, 1, sms, d);
    }
    return 0;
}
