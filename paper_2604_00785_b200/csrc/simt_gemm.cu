// Strided grouped GEMM on the CUDA cores: the fp32 path of the expert MLP.
//
// fp32 mode must agree with the fp32 CPU oracle within 1e-4 (BASELINE.json north
// star); TF32 tensor cores do not, so fp32 runs here. The k-loop is
// sequential in k with a separate multiply and add, i.e. the same accumulation
// order as the reference's grouped_mm / grouped_mm_nt / grouped_mm_weight_grad
// (include/optimus/kernels.hpp:111-189).
//
// D(g; m, n) (=|+=) scale * sum_k A(g; m, k) * B(g; k, n), every operand addressed by
// explicit element strides. Two grouping modes:
//   by_m: rows m are padded expert rows; the group of an m-tile comes from
//         group_start (multiples of kRowAlign); K and N are fixed.
//   by_k: one z-slice per group; the reduction runs over the group's rows
//         [group_start[g], group_start[g+1]); M and N are fixed.
#include "b2_common.cuh"
#include "kernels.h"

namespace b2 {

constexpr int kSBM = 64, kSBN = 64, kSBK = 16;

template <typename T>
__global__ void __launch_bounds__(256) simt_grouped_gemm_kernel(SimtGemmArgs a) {
    __shared__ float As[kSBK][kSBM + 1];
    __shared__ float Bs[kSBK][kSBN + 1];
    const T* A = static_cast<const T*>(a.A);
    const T* B = static_cast<const T*>(a.B);
    T* D = static_cast<T*>(a.D);
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
    const int n0 = blockIdx.y * kSBN;
    int g, m0, kbeg, kend;
    if (a.by_k) {
        g = blockIdx.z;
        m0 = blockIdx.x * kSBM;
        kbeg = a.group_start[g];
        kend = a.group_start[g + 1];
    } else {
        m0 = blockIdx.x * kSBM;
        if (m0 >= a.group_start[a.groups]) return;
        int lo = 0, hi = a.groups - 1;  // last g with group_start[g] <= m0
        while (lo < hi) {
            const int mid = (lo + hi + 1) / 2;
            if (a.group_start[mid] <= m0) lo = mid;
            else hi = mid - 1;
        }
        g = lo;
        kbeg = 0;
        kend = a.K;
    }
    const T* Ag = A + (int64_t)g * a.a_gs;
    const T* Bg = B + (int64_t)g * a.b_gs;
    float acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
    for (int k0 = kbeg; k0 < kend; k0 += kSBK) {
        for (int i = threadIdx.x; i < kSBK * kSBM; i += 256) {
            // consecutive threads walk the operand's contiguous dimension
            int kk, mm;
            if (a.lda_k == 1) { kk = i % kSBK; mm = i / kSBK; } else { mm = i % kSBM; kk = i / kSBM; }
            const int m = m0 + mm, k = k0 + kk;
            As[kk][mm] = (m < a.M_lim && k < kend) ? Elem<T>::load(Ag + (int64_t)m * a.lda_m + (int64_t)k * a.lda_k) : 0.f;
        }
        for (int i = threadIdx.x; i < kSBK * kSBN; i += 256) {
            int kk, nn;
            if (a.ldb_k == 1) { kk = i % kSBK; nn = i / kSBK; } else { nn = i % kSBN; kk = i / kSBN; }
            const int n = n0 + nn, k = k0 + kk;
            Bs[kk][nn] = (n < a.N && k < kend) ? Elem<T>::load(Bg + (int64_t)k * a.ldb_k + (int64_t)n * a.ldb_n) : 0.f;
        }
        __syncthreads();
        const int kn = min(kSBK, kend - k0);
        for (int kk = 0; kk < kn; ++kk) {
            float av[4], bv[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) av[i] = As[kk][ty * 4 + i];
#pragma unroll
            for (int j = 0; j < 4; ++j) bv[j] = Bs[kk][tx * 4 + j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = __fadd_rn(acc[i][j], __fmul_rn(av[i], bv[j]));
        }
        __syncthreads();
    }
    T* Dg = D + (int64_t)g * a.d_gs;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int m = m0 + ty * 4 + i;
        if (m >= a.M_lim) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int n = n0 + tx * 4 + j;
            if (n >= a.N) continue;
            T* dp = Dg + (int64_t)m * a.ldd_m + (int64_t)n * a.ldd_n;
            float v = acc[i][j];
            if (a.scale != 1.f) v = __fmul_rn(v, a.scale);
            if (a.accumulate) v = __fadd_rn(Elem<T>::to_f(*dp), v);
            *dp = Elem<T>::from_f(v);
        }
    }
}

template <typename T>
void launch_simt_grouped_gemm(const SimtGemmArgs& a, int64_t m_extent, cudaStream_t st) {
    if (m_extent <= 0 || a.N <= 0) return;
    dim3 grid((unsigned)ceil_div(m_extent, kSBM), (unsigned)ceil_div(a.N, kSBN), a.by_k ? (unsigned)a.groups : 1u);
    simt_grouped_gemm_kernel<T><<<grid, 256, 0, st>>>(a);
    B2_LAUNCH_CHECK();
}
template void launch_simt_grouped_gemm<float>(const SimtGemmArgs&, int64_t, cudaStream_t);
template void launch_simt_grouped_gemm<__nv_bfloat16>(const SimtGemmArgs&, int64_t, cudaStream_t);

}  // namespace b2
