// FP64 pipe throughput probe: independent DFMA chains, all SMs, event-timed.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_peak tools/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>
template <int CH>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
    double acc[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[c] = threadIdx.x * 1e-3 + c;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) acc[c] = fma(acc[c], a, b);
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += acc[c];
    if (s == 12345.678) out[0] = s;
}
__global__ void ffma_kernel(float* out, int iters, float a, float b) {
    float acc[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[c] = threadIdx.x * 1e-3f + c;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < 8; ++c) acc[c] = fmaf(acc[c], a, b);
    }
    float s = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) s += acc[c];
    if (s == 12345.678f) out[0] = s;
}
__global__ void f2f_kernel(float* out, int iters, float a) {
    float acc[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[c] = threadIdx.x * 1e-3f + c;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < 8; ++c) acc[c] = (float)((double)acc[c] * 0.5 + 0.25);  // F2F.F64.F32, DFMA, F2F.F32.F64
    }
    float s = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) s += acc[c];
    if (s == 12345.678f) out[0] = s;
}
int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* d;
    cudaMalloc(&d, 64);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 20000;
    for (int blocks_per_sm : {1, 2, 4, 8}) {
        const int grid = sms * blocks_per_sm, thr = 256;
        dfma_kernel<8><<<grid, thr>>>(d, 100, 0.999, 1e-3);
        cudaEventRecord(e0);
        dfma_kernel<8><<<grid, thr>>>(d, iters, 0.999, 1e-3);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double ops = (double)grid * thr * iters * 8;
        printf("DFMA %d blocks/SM x 256 thr: %.2f T DFMA/s = %.1f per clk per SM @1.965GHz\n", blocks_per_sm,
               ops / ms / 1e9, ops / ms / (sms * 1.965e6));
    }
    {
        const int grid = sms * 4, thr = 256;
        ffma_kernel<<<grid, thr>>>((float*)d, 100, 0.999f, 1e-3f);
        cudaEventRecord(e0);
        ffma_kernel<<<grid, thr>>>((float*)d, iters, 0.999f, 1e-3f);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double ops = (double)grid * thr * iters * 8;
        printf("FFMA: %.2f T FFMA/s = %.1f per clk per SM\n", ops / ms / 1e9, ops / ms / (sms * 1.965e6));
    }
    {
        const int grid = sms * 4, thr = 256;
        f2f_kernel<<<grid, thr>>>((float*)d, 100, 0.999f);
        cudaEventRecord(e0);
        f2f_kernel<<<grid, thr>>>((float*)d, iters, 0.999f);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double ops = (double)grid * thr * iters * 8;
        printf("F2F f32->f64 + DFMA + F2F f64->f32 chains: %.2f T/s = %.2f per clk per SM (each of 3 ops)\n", ops / ms / 1e9,
               ops / ms / (sms * 1.965e6));
    }
    return 0;
}
