// Permute / unpermute between token-major tensors and the expert-sorted, 128-row
// padded row space the grouped GEMMs work in, plus the element-wise SwiGLU pieces
// used by the fp32 (SIMT) path.
//
// Reference: row gather in expert_forward (include/optimus/moe.hpp:229-232),
// output_reduction_forward (moe.hpp:250-268), output_reduction_backward
// (moe.hpp:271-298), the scatter-add to gathered tokens (moe.hpp:418-423) plus the
// router input-gradient term (moe.hpp:454, matmul_nt kernels.hpp:75-96), silu_glu /
// silu_glu_backward (kernels.hpp:262-295).
//
// All kernels are deterministic: every output element is produced by exactly one
// thread, summing in the reference's slot (k) order; no atomics. Row-copy kernels
// move 16-byte vectors (one warp per row) when H*sizeof(T) allows.
#include "b2_common.cuh"
#include "kernels.h"

namespace b2 {

template <typename T>
__device__ __forceinline__ bool vec_ok(int H) {
    return ((int64_t)H * (int64_t)sizeof(T)) % 16 == 0;
}

// mlp_in[prow] = x[prow_src[prow]] (zero row when prow_src < 0); rows < *p_total
template <typename T>
__global__ void gather_rows_kernel(const T* __restrict__ x, const int32_t* __restrict__ prow_src,
                                   const int32_t* __restrict__ p_total, T* __restrict__ out, int H, int64_t pmax) {
    const int64_t P = min((int64_t)*p_total, pmax);
    const int lane = threadIdx.x % 32;
    const int64_t warps = (int64_t)gridDim.x * blockDim.x / 32;
    for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32; r < P; r += warps) {
        const int src = prow_src[r];
        T* dst = out + r * H;
        if (vec_ok<T>(H)) {
            const int nv = (int)((int64_t)H * sizeof(T) / 16);
            int4* d4 = reinterpret_cast<int4*>(dst);
            if (src < 0) {
                for (int v = lane; v < nv; v += 32) d4[v] = make_int4(0, 0, 0, 0);
            } else {
                const int4* s4 = reinterpret_cast<const int4*>(x + (int64_t)src * H);
                for (int v = lane; v < nv; v += 32) d4[v] = __ldg(s4 + v);
            }
        } else {
            for (int c = lane; c < H; c += 32) dst[c] = src < 0 ? Elem<T>::from_f(0.f) : x[(int64_t)src * H + c];
        }
    }
}

// zero the pad rows of a padded buffer (rows < *p_total whose prow_src < 0)
template <typename T>
__global__ void zero_pad_rows_kernel(T* __restrict__ buf, const int32_t* __restrict__ prow_src,
                                     const int32_t* __restrict__ p_total, int W, int64_t pmax) {
    const int64_t P = min((int64_t)*p_total, pmax);
    const int lane = threadIdx.x % 32;
    const int64_t warps = (int64_t)gridDim.x * blockDim.x / 32;
    for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32; r < P; r += warps) {
        if (prow_src[r] >= 0) continue;
        for (int c = lane; c < W; c += 32) buf[r * W + c] = Elem<T>::from_f(0.f);
    }
}

// out[t, c] = sum over t's local slots j (in order) of weights[t, selected_k[j]] * y[slot_prow[j], c]
// (moe.hpp:258-266, T arithmetic: multiply, then add)
template <typename T>
__global__ void combine_kernel(const T* __restrict__ y, const int32_t* __restrict__ slot_prow,
                               const int32_t* __restrict__ selected_k, const int32_t* __restrict__ cum_expert_counts,
                               const float* __restrict__ gw, T* __restrict__ out, int T_tok, int H, int K) {
    const int t = (blockIdx.x * blockDim.x + threadIdx.x) / 32, lane = threadIdx.x % 32;
    if (t >= T_tok) return;
    const int j0 = cum_expert_counts[t], j1 = cum_expert_counts[t + 1];
    for (int c0 = lane * 4; c0 < H; c0 += 128) {
        float acc[4] = {0.f, 0.f, 0.f, 0.f};
        for (int j = j0; j < j1; ++j) {
            const float wv = gw[(int64_t)t * K + selected_k[j]];
            const T* yr = y + (int64_t)slot_prow[j] * H;
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (c0 + q < H) acc[q] = __fadd_rn(acc[q], __fmul_rn(wv, Elem<T>::to_f(yr[c0 + q])));
        }
#pragma unroll
        for (int q = 0; q < 4; ++q)
            if (c0 + q < H) out[(int64_t)t * H + c0 + q] = Elem<T>::from_f(acc[q]);
    }
}

// output_reduction_backward (moe.hpp:271-298): for each local slot of token t,
// dy[prow] = w * dout[t]; wgrad[t, k] = <dout[t], y[prow]> accumulated in fp64.
// Non-local (t, k) entries of wgrad are written as 0.
template <typename T>
__global__ void out_reduction_bwd_kernel(const T* __restrict__ dout, const T* __restrict__ y,
                                         const int32_t* __restrict__ slot_prow, const int32_t* __restrict__ selected_k,
                                         const int32_t* __restrict__ cum_expert_counts, const float* __restrict__ gw,
                                         T* __restrict__ dy, float* __restrict__ wgrad, int T_tok, int H, int K) {
    const int t = (blockIdx.x * blockDim.x + threadIdx.x) / 32, lane = threadIdx.x % 32;
    if (t >= T_tok) return;
    const int j0 = cum_expert_counts[t], j1 = cum_expert_counts[t + 1];
    for (int k = lane; k < K; k += 32) wgrad[(int64_t)t * K + k] = 0.f;
    __syncwarp();
    const T* gp = dout + (int64_t)t * H;
    for (int j = j0; j < j1; ++j) {
        const int k = selected_k[j];
        const int64_t r = slot_prow[j];
        const float wv = gw[(int64_t)t * K + k];
        double dot = 0.0;
        for (int c = lane; c < H; c += 32) {
            const float g = Elem<T>::to_f(gp[c]);
            dy[r * H + c] = Elem<T>::from_f(__fmul_rn(wv, g));
            dot += (double)g * (double)Elem<T>::to_f(y[r * H + c]);
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
        if (lane == 0) wgrad[(int64_t)t * K + k] = (float)dot;
    }
}

// dx[t, h] = (sum over t's slots of dxp[slot_prow, h]) [or base[t, h]] + sum_e dl[t, e] * Wr[h, e]
// 64 tokens x 64 h per CTA; the router term is a small SIMT GEMM (matmul_nt order).
constexpr int kDxT = 64, kDxH = 64, kDxE = 32;
template <typename T, bool FROM_SLOTS>
__global__ void __launch_bounds__(256) dx_finalize_kernel(const T* __restrict__ src, const int32_t* __restrict__ slot_prow,
                                                          const int32_t* __restrict__ cum_expert_counts,
                                                          const float* __restrict__ dl, const T* __restrict__ wr,
                                                          T* __restrict__ dx, int S, int H, int N) {
    __shared__ float ds[kDxE][kDxT + 1];
    __shared__ float ws[kDxE][kDxH + 1];
    const int t0 = blockIdx.x * kDxT, h0 = blockIdx.y * kDxH;
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
    float acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
    for (int e0 = 0; e0 < N; e0 += kDxE) {
        for (int i = threadIdx.x; i < kDxE * kDxT; i += 256) {
            const int ee = i % kDxE, tt = i / kDxE;
            const int e = e0 + ee, t = t0 + tt, h = h0 + tt;
            ds[ee][tt] = (e < N && t < S) ? dl[(int64_t)t * N + e] : 0.f;
            ws[ee][tt] = (e < N && h < H) ? Elem<T>::load(wr + (int64_t)h * N + e) : 0.f;
        }
        __syncthreads();
        const int eend = min(kDxE, N - e0);
        for (int ee = 0; ee < eend; ++ee) {
            float a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = ds[ee][ty * 4 + i];
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = ws[ee][tx * 4 + j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = __fadd_rn(acc[i][j], __fmul_rn(a[i], b[j]));
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int t = t0 + ty * 4 + i;
        if (t >= S) continue;
        int j0 = 0, j1 = 0;
        if (FROM_SLOTS) {
            j0 = cum_expert_counts[t];
            j1 = cum_expert_counts[t + 1];
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int h = h0 + tx * 4 + j;
            if (h >= H) continue;
            float base = 0.f;
            if (FROM_SLOTS) {
                for (int s = j0; s < j1; ++s) base = __fadd_rn(base, Elem<T>::to_f(src[(int64_t)slot_prow[s] * H + h]));
            } else {
                base = Elem<T>::to_f(src[(int64_t)t * H + h]);
            }
            dx[(int64_t)t * H + h] = Elem<T>::from_f(__fadd_rn(base, acc[i][j]));
        }
    }
}

// ---- element-wise SwiGLU (kernels.hpp:262-295), fp64 math in fp32 mode ------------------

template <typename W>
__device__ __forceinline__ W silu_w(W x) {
    return x / (W(1) + exp(-x));
}

template <typename T>
__global__ void swiglu_fwd_kernel(const T* __restrict__ g, const T* __restrict__ u, T* __restrict__ h,
                                  const int32_t* __restrict__ p_total, int I, int64_t pmax) {
    using W = typename Elem<T>::Wide;
    const int64_t n = min((int64_t)*p_total, pmax) * I;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const W x = (W)Elem<T>::to_f(g[i]);
        h[i] = Elem<T>::from_f((float)(silu_w<W>(x) * (W)Elem<T>::to_f(u[i])));
    }
}

// dgu row layout: [dgate (I) | dup (I)]
template <typename T>
__global__ void swiglu_bwd_kernel(const T* __restrict__ g, const T* __restrict__ u, const T* __restrict__ dh,
                                  T* __restrict__ dgu, const int32_t* __restrict__ p_total, int I, int64_t pmax) {
    using W = typename Elem<T>::Wide;
    const int64_t n = min((int64_t)*p_total, pmax) * I;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / I, c = i % I;
        const W x = (W)Elem<T>::to_f(g[i]);
        const W d = (W)Elem<T>::to_f(dh[i]);
        const W s = W(1) / (W(1) + exp(-x));
        const W dsilu = s * (W(1) + x * (W(1) - s));
        dgu[r * 2 * I + I + c] = Elem<T>::from_f((float)(silu_w<W>(x) * d));
        dgu[r * 2 * I + c] = Elem<T>::from_f((float)((W)Elem<T>::to_f(u[i]) * d * dsilu));
    }
}

// ---- launchers ------------------------------------------------------------------------

static unsigned grid_for_rows(int64_t pmax) { return (unsigned)std::max<int64_t>(1, std::min<int64_t>(148 * 16, ceil_div(pmax, 8))); }

template <typename T>
void launch_gather_rows(const T* x, const int32_t* prow_src, const int32_t* p_total, T* out, int H, int64_t pmax,
                        cudaStream_t st) {
    if (pmax <= 0) return;
    gather_rows_kernel<T><<<grid_for_rows(pmax), 256, 0, st>>>(x, prow_src, p_total, out, H, pmax);
    B2_LAUNCH_CHECK();
}

template <typename T>
void launch_zero_pad_rows(T* buf, const int32_t* prow_src, const int32_t* p_total, int W, int64_t pmax,
                          cudaStream_t st) {
    if (pmax <= 0) return;
    zero_pad_rows_kernel<T><<<grid_for_rows(pmax), 256, 0, st>>>(buf, prow_src, p_total, W, pmax);
    B2_LAUNCH_CHECK();
}

template <typename T>
void launch_combine(const T* y, const int32_t* slot_prow, const int32_t* selected_k, const int32_t* cec,
                    const float* gw, T* out, int T_tok, int H, int K, cudaStream_t st) {
    if (T_tok <= 0) return;
    combine_kernel<T><<<(unsigned)ceil_div(T_tok, 8), 256, 0, st>>>(y, slot_prow, selected_k, cec, gw, out, T_tok, H, K);
    B2_LAUNCH_CHECK();
}

template <typename T>
void launch_out_reduction_bwd(const T* dout, const T* y, const int32_t* slot_prow, const int32_t* selected_k,
                              const int32_t* cec, const float* gw, T* dy, float* wgrad, int T_tok, int H, int K,
                              cudaStream_t st) {
    if (T_tok <= 0) return;
    out_reduction_bwd_kernel<T><<<(unsigned)ceil_div(T_tok, 8), 256, 0, st>>>(dout, y, slot_prow, selected_k, cec, gw,
                                                                               dy, wgrad, T_tok, H, K);
    B2_LAUNCH_CHECK();
}

template <typename T>
void launch_dx_finalize(const T* src, bool from_slots, const int32_t* slot_prow, const int32_t* cec, const float* dl,
                        const T* wr, T* dx, int S, int H, int N, cudaStream_t st) {
    if (S <= 0) return;
    dim3 grid((unsigned)ceil_div(S, kDxT), (unsigned)ceil_div(H, kDxH));
    if (from_slots)
        dx_finalize_kernel<T, true><<<grid, 256, 0, st>>>(src, slot_prow, cec, dl, wr, dx, S, H, N);
    else
        dx_finalize_kernel<T, false><<<grid, 256, 0, st>>>(src, slot_prow, cec, dl, wr, dx, S, H, N);
    B2_LAUNCH_CHECK();
}

template <typename T>
void launch_swiglu_fwd(const T* g, const T* u, T* h, const int32_t* p_total, int I, int64_t pmax, cudaStream_t st) {
    if (pmax <= 0) return;
    swiglu_fwd_kernel<T><<<148 * 8, 256, 0, st>>>(g, u, h, p_total, I, pmax);
    B2_LAUNCH_CHECK();
}

template <typename T>
void launch_swiglu_bwd(const T* g, const T* u, const T* dh, T* dgu, const int32_t* p_total, int I, int64_t pmax,
                       cudaStream_t st) {
    if (pmax <= 0) return;
    swiglu_bwd_kernel<T><<<148 * 8, 256, 0, st>>>(g, u, dh, dgu, p_total, I, pmax);
    B2_LAUNCH_CHECK();
}

#define B2_INST(T)                                                                                              \
    template void launch_gather_rows<T>(const T*, const int32_t*, const int32_t*, T*, int, int64_t, cudaStream_t); \
    template void launch_zero_pad_rows<T>(T*, const int32_t*, const int32_t*, int, int64_t, cudaStream_t);        \
    template void launch_combine<T>(const T*, const int32_t*, const int32_t*, const int32_t*, const float*, T*, int, \
                                    int, int, cudaStream_t);                                                       \
    template void launch_out_reduction_bwd<T>(const T*, const T*, const int32_t*, const int32_t*, const int32_t*,   \
                                              const float*, T*, float*, int, int, int, cudaStream_t);              \
    template void launch_dx_finalize<T>(const T*, bool, const int32_t*, const int32_t*, const float*, const T*, T*, \
                                        int, int, int, cudaStream_t);                                              \
    template void launch_swiglu_fwd<T>(const T*, const T*, T*, const int32_t*, int, int64_t, cudaStream_t);        \
    template void launch_swiglu_bwd<T>(const T*, const T*, const T*, T*, const int32_t*, int, int64_t, cudaStream_t);
B2_INST(float)
B2_INST(__nv_bfloat16)
#undef B2_INST

}  // namespace b2
