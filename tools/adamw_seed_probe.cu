// Max relative error of the fp64 MUFU seeds the AdamW fast path starts from (adamw.cu):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/adamw_seed_probe.cu -o build/probe/seed_err
// 8 G inputs with exponents in [2^-120, 2^120] (the fast path's guarded range).
#include <cstdio>
#include <cstdint>
__global__ void k(double* out, uint64_t n, uint64_t seed) {
    double mr = 0, mq = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t x = (i + seed) * 0x9E3779B97F4A7C15ull; x ^= x >> 29; x *= 0xBF58476D1CE4E5B9ull; x ^= x >> 32;
        // exponents in [2^-120, 2^120]
        uint64_t e = 1023 - 120 + (x % 241);
        double d = __longlong_as_double((long long)((e << 52) | ((x * 0x94D049BB133111EBull) >> 12)));
        double y, r;
        asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
        asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
        double ey = fabs(__fma_rn(y * y, d, -1.0)) * 0.5;  // rel err of y ~ (y^2 d - 1)/2
        double er = fabs(__fma_rn(r, d, -1.0));
        mr = fmax(mr, ey); mq = fmax(mq, er);
    }
    atomicMax((unsigned long long*)&out[0], (unsigned long long)__double_as_longlong(mr));
    atomicMax((unsigned long long*)&out[1], (unsigned long long)__double_as_longlong(mq));
}
int main() {
    double* d; cudaMalloc(&d, 16); cudaMemset(d, 0, 16);
    for (int s = 0; s < 8; ++s) k<<<1184, 256>>>(d, 1ull << 30, s * (1ull << 30));
    double h[2]; cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("max rel err: rsqrt.approx.f64 %.3e (2^%.2f), rcp.approx.f64 %.3e (2^%.2f)\n", h[0], log2(h[0]), h[1], log2(h[1]));
}
