// Fused optimizer-shard kernels: grad unscale (+ clip) -> AdamW -> bf16 recast.
//
// Reference: adamw_update (src/optim.cpp:88-107) and the per-slice steps of
// ShardedOptimizer::step (optim.cpp:155 mean scale, 160-166 norm, 168-178 clip).
// The arithmetic is the reference's, in fp64 with fp32-rounded moments, written
// with explicit _rn intrinsics so nvcc cannot contract it into FMAs: given the same
// inputs the master, moments and the bf16 weight are bitwise identical to the CPU.
// HBM traffic per element: grad 2-4 B + master/m/v 12 B in + 12 B out + weight 2-4 B.
#include <cstdlib>
#include <string>

#include "b2_common.cuh"
#include "kernels.h"

namespace b2 {

__device__ __forceinline__ float load_grad(const void* g, int dtype, int64_t i) {
    return dtype == F32 ? static_cast<const float*>(g)[i]
                        : __bfloat162float(static_cast<const __nv_bfloat16*>(g)[i]);
}

// bf16 round-to-nearest-even of the master (common.hpp:116-131), NaN kept quiet
__device__ __forceinline__ uint16_t bf16_bits_rne(float f) {
    const uint32_t u = __float_as_uint(f);
    if (isnan(f)) return (uint16_t)((u >> 16) | 0x0040u);
    return (uint16_t)((u + 0x7fffu + ((u >> 16) & 1u)) >> 16);
}

struct AdamWDev {
    double lr, b1, b2, omb1, omb2, eps, lr_wd, bc1, bc2;
    double rbc1, rbc2;  // RN(1/bc1), RN(1/bc2), computed on the host
    double lr_rbc1;     // lr * rbc1 (the fast path's estimate only)
};

// a / b, correctly rounded, for the step constants b = bc1, bc2 with y = RN(1/b): q0 = a*y is
// within 1.5 ulp, one remainder correction makes it faithful and the second one (Markstein's
// theorem: exact remainder fma(-b, q, a), correctly rounded reciprocal) rounds it correctly.
// 5 DFMA/DMUL and no slow-path branch, instead of __ddiv_rn's reciprocal refinement.
__device__ __forceinline__ double div_const(double a, double b, double y) {
    const double q0 = __dmul_rn(a, y);
    const double q1 = __fma_rn(__fma_rn(-b, q0, a), y, q0);
    const double q2 = __fma_rn(__fma_rn(-b, q1, a), y, q1);
    // branch-free (selects): +-0 / b = +-0 = a; inf / b = inf * y (b > 0); NaN propagates
    return a == 0.0 ? a : (isfinite(a) ? q2 : q0);
}

// The update term U = RN(RN(lr * RN(m / bc1)) / RN(RN(sqrt(RN(v / bc2))) + eps)) in the
// reference's correctly rounded steps (div_const, __dsqrt_rn, __ddiv_rn).
__device__ __forceinline__ double update_exact(double md, double vd, const AdamWDev& c) {
    const double num = __dmul_rn(c.lr, div_const(md, c.bc1, c.rbc1));
    const double den = __dadd_rn(__dsqrt_rn(div_const(vd, c.bc2, c.rbc2)), c.eps);
    return __ddiv_rn(num, den);
}

// Fast path with an exactness certificate. U' comes from the MUFU rsqrt / rcp seeds of the fp64
// values (rsqrt.approx.f64 / rcp.approx.f64: measured within 2^-19.9, tools/adamw_seed_probe.cu)
// and one fp64 Newton step each, so |U' - U| <= 2^-36 |U| even for seeds 2x worse (the step
// squares the seed error; ~12 fp64 roundings and the reference's own 6 ulp add 2^-49). Hence
// W1 - U lies within tol = 2^-30 |U'| + 2^-50 |W'| of W' = W1 - U' (margins 64x / 4x). Float
// rounding is monotonic: when W' - tol and W' + tol round to the same float, so does W1 - U,
// and that float is the reference's master. Otherwise (W' within tol of a rounding boundary:
// ~1e-4 of the elements at training scale) and for inputs outside the seeds' normal range,
// non-finite values included, the exact sequence runs — bitwise the reference's either way.
// Against the exact sequence alone: 0.59 -> 0.37 G fp64 instructions per 0.5 G elements and
// 5.59-5.70 -> 5.25-5.29 ms per G elements (tools/adamw_probe.py), where a kernel with the
// same loads and stores and no fp64 math takes 5.08 ms.
__device__ __forceinline__ void adamw_elem(float& master, float& m, float& v, float g, const AdamWDev& c,
                                           float& wout_f) {
    double w = (double)master;
    const double gd = (double)g;
    w = __dsub_rn(w, __dmul_rn(c.lr_wd, w));                                       // w -= lr*wd*w
    const double mm = __dadd_rn(__dmul_rn(c.b1, (double)m), __dmul_rn(c.omb1, gd));  // b1*m + (1-b1)*g
    const double vv = __dadd_rn(__dmul_rn(c.b2, (double)v), __dmul_rn(__dmul_rn(c.omb2, gd), gd));
    m = (float)mm;
    v = (float)vv;
    const double md = (double)m, vd = (double)v;
    const double np = __dmul_rn(md, c.lr_rbc1);  // ~ lr * (m / bc1)
    const double bp = __dmul_rn(vd, c.rbc2);     // ~ v / bc2
    double y0, r0;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y0) : "d"(bp));
    const double s0 = __dmul_rn(bp, y0);
    const double sq = __fma_rn(__fma_rn(-s0, s0, bp), __dmul_rn(0.5, y0), s0);  // ~ sqrt(v / bc2)
    const double den = __dadd_rn(sq, c.eps);
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r0) : "d"(den));
    const double q0 = __dmul_rn(np, r0);
    // m == +-0 with a positive denominator (v > 0, or v == 0 and eps > 0): U = +-0 exactly, with
    // m's sign, which matters when W1 is a zero too
    const bool mzero = md == 0.0 && (vd > 0.0 || (vd == 0.0 && c.eps > 0.0));
    const double up = mzero ? np : __fma_rn(__fma_rn(-den, q0, np), r0, q0);
    const double wn = __dsub_rn(w, up);
    const double tol = __fma_rn(fabs(up), 0x1p-30, __dmul_rn(fabs(wn), 0x1p-50));
    const float lo = __double2float_rn(__dsub_rn(wn, tol)), hi = __double2float_rn(__dadd_rn(wn, tol));
    const bool ok = mzero || (bp >= 0x1p-120 && bp <= 0x1p120 && __float_as_uint(lo) == __float_as_uint(hi));
    if (__builtin_expect(ok, 1)) {
        master = mzero ? (float)wn : lo;
    } else {
        master = (float)__dsub_rn(w, update_exact(md, vd, c));
    }
    wout_f = master;
}

// grad_scale: the (float)(1/g) of optim.cpp:155; the clip scale is derived on the
// device from the global norm (optim.cpp:168-171) so the step never waits on the host.
__global__ void adamw_kernel(float* __restrict__ master, float* __restrict__ mom, float* __restrict__ vel,
                             const void* __restrict__ grad, int grad_dtype, void* __restrict__ wout, int wdtype,
                             int64_t n, AdamWDev c, float grad_scale, const double* __restrict__ norm_sq,
                             double clip_norm, int clip_active, int round_bf16) {
    double clip = 1.0;
    if (norm_sq) {
        const double norm = sqrt(*norm_sq);
        if (clip_active && norm > clip_norm && norm > 0) clip = clip_norm / norm;
    }
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        float g = load_grad(grad, grad_dtype, i);
        if (grad_scale != 1.f) g = __fmul_rn(g, grad_scale);
        if (clip != 1.0) g = (float)__dmul_rn((double)g, clip);
        float ms = master[i], mv = mom[i], vv = vel[i], wf;
        adamw_elem(ms, mv, vv, g, c, wf);
        master[i] = ms;
        mom[i] = mv;
        vel[i] = vv;
        if (wdtype == F32) {
            static_cast<float*>(wout)[i] = round_bf16 ? __uint_as_float((uint32_t)bf16_bits_rne(wf) << 16) : wf;
        } else {
            static_cast<uint16_t*>(wout)[i] = bf16_bits_rne(wf);
        }
    }
}

// vectorised fast path: bf16 grads, bf16 weights; each thread-iteration handles two
// groups of 4 elements with all 8 loads issued before the fp64 math (more bytes in flight)
__device__ __forceinline__ void adamw_group4(float4& ms, float4& mv, float4& vv, uint2 gb, const AdamWDev& c,
                                             float grad_scale, double clip, uint2& wout) {
    float g[4] = {__uint_as_float(gb.x << 16), __uint_as_float(gb.x & 0xFFFF0000u), __uint_as_float(gb.y << 16),
                  __uint_as_float(gb.y & 0xFFFF0000u)};
    float* pm = &ms.x;
    float* pv1 = &mv.x;
    float* pv2 = &vv.x;
    uint16_t wb[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        float gq = g[q];
        if (grad_scale != 1.f) gq = __fmul_rn(gq, grad_scale);
        if (clip != 1.0) gq = (float)__dmul_rn((double)gq, clip);
        float wf;
        adamw_elem(pm[q], pv1[q], pv2[q], gq, c, wf);
        wb[q] = bf16_bits_rne(wf);
    }
    wout = make_uint2((uint32_t)wb[0] | ((uint32_t)wb[1] << 16), (uint32_t)wb[2] | ((uint32_t)wb[3] << 16));
}

__global__ void __launch_bounds__(256) adamw_bf16x4_kernel(float4* __restrict__ master, float4* __restrict__ mom,
                                                           float4* __restrict__ vel, const uint2* __restrict__ grad,
                                                           uint2* __restrict__ wout, int64_t n4, AdamWDev c,
                                                           float grad_scale, const double* __restrict__ norm_sq,
                                                           double clip_norm, int clip_active) {
    double clip = 1.0;
    if (norm_sq) {
        const double norm = sqrt(*norm_sq);
        if (clip_active && norm > clip_norm && norm > 0) clip = clip_norm / norm;
    }
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + stride < n4; i += 2 * stride) {
        const int64_t j = i + stride;
        const uint2 g0 = __ldcs(grad + i), g1 = __ldcs(grad + j);
        float4 m0 = __ldcs(master + i), a0 = __ldcs(mom + i), v0 = __ldcs(vel + i);
        float4 m1 = __ldcs(master + j), a1 = __ldcs(mom + j), v1 = __ldcs(vel + j);
        uint2 w0, w1;
        adamw_group4(m0, a0, v0, g0, c, grad_scale, clip, w0);
        adamw_group4(m1, a1, v1, g1, c, grad_scale, clip, w1);
        __stcs(master + i, m0);
        __stcs(mom + i, a0);
        __stcs(vel + i, v0);
        __stcs(wout + i, w0);
        __stcs(master + j, m1);
        __stcs(mom + j, a1);
        __stcs(vel + j, v1);
        __stcs(wout + j, w1);
    }
    if (i < n4) {
        const uint2 g0 = __ldcs(grad + i);
        float4 m0 = __ldcs(master + i), a0 = __ldcs(mom + i), v0 = __ldcs(vel + i);
        uint2 w0;
        adamw_group4(m0, a0, v0, g0, c, grad_scale, clip, w0);
        __stcs(master + i, m0);
        __stcs(mom + i, a0);
        __stcs(vel + i, v0);
        __stcs(wout + i, w0);
    }
}

// sum of squares of the scaled slice, fp64, fixed-order block reduction, then
// accumulated into *acc in launch order (deterministic)
__global__ void sumsq_partial_kernel(const void* __restrict__ g, int dtype, int64_t n, float scale,
                                     double* __restrict__ partials) {
    double s = 0.0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        float v = load_grad(g, dtype, i);
        if (scale != 1.f) v = __fmul_rn(v, scale);
        s += (double)v * (double)v;
    }
    __shared__ double red[256];
    red[threadIdx.x] = s;
    __syncthreads();
    for (int o = blockDim.x / 2; o; o >>= 1) {
        if ((int)threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) partials[blockIdx.x] = red[0];
}

__global__ void sumsq_final_kernel(const double* __restrict__ partials, int nparts, double* __restrict__ acc,
                                   int init) {
    if (threadIdx.x != 0) return;
    double s = 0.0;
    for (int i = 0; i < nparts; ++i) s += partials[i];
    *acc = init ? s : *acc + s;
}

static int adamw_grid(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>(148 * 8, ceil_div(n, 256))); }

void launch_adamw_full(const AdamWKernelArgs& a, const double* norm_sq, double clip_norm, int clip_active,
                       cudaStream_t st) {
    if (a.n <= 0) return;
    AdamWDev c;
    c.lr = a.lr;
    c.b1 = a.beta1;
    c.b2 = a.beta2;
    c.omb1 = 1.0 - a.beta1;
    c.omb2 = 1.0 - a.beta2;
    c.eps = a.eps;
    c.lr_wd = a.lr * a.weight_decay;
    c.bc1 = a.bc1;
    c.bc2 = a.bc2;
    c.rbc1 = 1.0 / a.bc1;
    c.rbc2 = 1.0 / a.bc2;
    c.lr_rbc1 = a.lr * c.rbc1;
    const float gs = (float)a.grad_scale;
    const bool vec = a.grad_dtype == BF16 && a.weight_dtype == BF16 && a.round_bf16 && a.n % 4 == 0 &&
                     ((uintptr_t)a.master % 16 == 0) && ((uintptr_t)a.m % 16 == 0) && ((uintptr_t)a.v % 16 == 0) &&
                     ((uintptr_t)a.grad % 8 == 0) && ((uintptr_t)a.weight_out % 8 == 0);
    if (vec) {
        adamw_bf16x4_kernel<<<adamw_grid(a.n / 4), 256, 0, st>>>((float4*)a.master, (float4*)a.m, (float4*)a.v,
                                                                 (const uint2*)a.grad, (uint2*)a.weight_out, a.n / 4,
                                                                 c, gs, norm_sq, clip_norm, clip_active);
    } else {
        adamw_kernel<<<adamw_grid(a.n), 256, 0, st>>>(a.master, a.m, a.v, a.grad, a.grad_dtype, a.weight_out,
                                                      a.weight_dtype, a.n, c, gs, norm_sq, clip_norm, clip_active,
                                                      a.round_bf16);
    }
    B2_LAUNCH_CHECK();
}

void launch_adamw(const AdamWKernelArgs& a, cudaStream_t st) { launch_adamw_full(a, nullptr, 0.0, 0, st); }

void launch_sumsq_acc(const void* g, int dtype, int64_t n, float scale, double* partials, int nparts, double* acc,
                      bool init, cudaStream_t st) {
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(nparts, ceil_div(std::max<int64_t>(n, 1), 256)));
    sumsq_partial_kernel<<<grid, 256, 0, st>>>(g, dtype, n, scale, partials);
    B2_LAUNCH_CHECK();
    sumsq_final_kernel<<<1, 32, 0, st>>>(partials, grid, acc, init ? 1 : 0);
    B2_LAUNCH_CHECK();
}

void launch_sumsq(const void* g, int dtype, int64_t n, double scale, double* partials, int nparts, cudaStream_t st) {
    launch_sumsq_acc(g, dtype, n, (float)scale, partials, nparts, partials + nparts, true, st);
}

__global__ void scale_to_f32_kernel(const void* __restrict__ src, int dtype, int64_t n, float scale,
                                    float* __restrict__ dst) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = __fmul_rn(load_grad(src, dtype, i), scale);
}

void launch_scale_to_f32(const void* src, int dtype, int64_t n, double scale, float* dst, cudaStream_t st) {
    if (n <= 0) return;
    scale_to_f32_kernel<<<adamw_grid(n), 256, 0, st>>>(src, dtype, n, (float)scale, dst);
    B2_LAUNCH_CHECK();
}

__global__ void scale_inplace_kernel(void* __restrict__ buf, int dtype, int64_t n, float scale) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        if (dtype == F32) {
            float* p = static_cast<float*>(buf);
            p[i] = __fmul_rn(p[i], scale);
        } else {
            __nv_bfloat16* p = static_cast<__nv_bfloat16*>(buf);
            p[i] = __float2bfloat16_rn(__fmul_rn(__bfloat162float(p[i]), scale));
        }
    }
}

void launch_scale_inplace(void* buf, int dtype, int64_t n, float scale, cudaStream_t st) {
    if (n <= 0) return;
    scale_inplace_kernel<<<adamw_grid(n), 256, 0, st>>>(buf, dtype, n, scale);
    B2_LAUNCH_CHECK();
}

// ---------------------------------------------------------------- multi-tensor step

__device__ __forceinline__ void flag_nonfinite(bool bad, int32_t* flag) {
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x % 32) == 0) atomicExch(flag, 1);
}

__device__ __forceinline__ double block_sum_fixed(double s, double* red) {
    red[threadIdx.x] = s;
    __syncthreads();
    for (int o = blockDim.x / 2; o; o >>= 1) {
        if ((int)threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
        __syncthreads();
    }
    return red[0];
}

__global__ void __launch_bounds__(256) sumsq_chunks_kernel(const OptSeg* __restrict__ segs,
                                                           const OptChunk* __restrict__ chunks,
                                                           const int32_t* __restrict__ ids, int grad_dtype,
                                                           double* __restrict__ partials, int32_t* nonfinite) {
    pdl_wait();
    pdl_launch();
    __shared__ double red[256];
    const int cid = ids[blockIdx.x];
    const OptChunk ch = chunks[cid];
    const OptSeg sg = segs[ch.seg];
    const float scale = sg.scale;
    double s = 0.0;
    bool bad = false;
    if (grad_dtype == BF16 && (ch.begin % 8) == 0 &&
        (((uintptr_t)sg.grad + 2 * ch.begin) & 15) == 0) {
        const uint4* g8 = reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(sg.grad) + ch.begin);
        const int64_t n8 = ch.len / 8;
        for (int64_t i = threadIdx.x; i < n8; i += blockDim.x) {
            const uint4 r = __ldcs(g8 + i);
            const uint32_t w[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                float a = __uint_as_float(w[q] << 16), b = __uint_as_float(w[q] & 0xFFFF0000u);
                if (scale != 1.f) {
                    a = __fmul_rn(a, scale);
                    b = __fmul_rn(b, scale);
                }
                bad |= !isfinite(a) || !isfinite(b);
                s += (double)a * (double)a;
                s += (double)b * (double)b;
            }
        }
        for (int64_t i = 8 * n8 + threadIdx.x; i < ch.len; i += blockDim.x) {
            float v = load_grad(sg.grad, grad_dtype, ch.begin + i);
            if (scale != 1.f) v = __fmul_rn(v, scale);
            bad |= !isfinite(v);
            s += (double)v * (double)v;
        }
    } else {
        for (int64_t i = threadIdx.x; i < ch.len; i += blockDim.x) {
            float v = load_grad(sg.grad, grad_dtype, ch.begin + i);
            if (scale != 1.f) v = __fmul_rn(v, scale);
            bad |= !isfinite(v);
            s += (double)v * (double)v;
        }
    }
    flag_nonfinite(bad, nonfinite);
    const double tot = block_sum_fixed(s, red);
    if (threadIdx.x == 0) partials[cid] = tot;
}

__global__ void __launch_bounds__(1024) norm_final_kernel(const double* __restrict__ partials, int n,
                                                          double* __restrict__ out) {
    pdl_wait();
    pdl_launch();
    __shared__ double red[1024];
    const int per = (n + blockDim.x - 1) / blockDim.x;
    double s = 0.0;
    const int b = threadIdx.x * per, e = min(n, b + per);
    for (int i = b; i < e; ++i) s += partials[i];
    const double tot = block_sum_fixed(s, red);
    if (threadIdx.x == 0) *out = tot;
}

// 256 threads x 4 blocks per SM: the fp64 divide / sqrt chains are long, so occupancy (not the
// FP64 pipe, ~28 % busy at 3 blocks) is what keeps enough bytes in flight
template <int MINB>
__global__ void __launch_bounds__(256, MINB) adamw_chunks_kernel(const OptSeg* __restrict__ segs,
                                                           const OptChunk* __restrict__ chunks,
                                                           const int32_t* __restrict__ ids, int nids, AdamWDev c,
                                                           OptStepArgs a, const double* __restrict__ norm_sq) {
    pdl_wait();
    pdl_launch();
    double clip = 1.0;
    if (norm_sq) {
        const double norm = sqrt(*norm_sq);
        if (a.clip_active && norm > a.clip_norm && norm > 0) clip = a.clip_norm / norm;
    }
    for (int q = blockIdx.x; q < nids; q += gridDim.x) {
        const OptChunk ch = chunks[ids[q]];
        const OptSeg sg = segs[ch.seg];
        if (sg.vec) {
            float4* ms = reinterpret_cast<float4*>(sg.master + ch.begin);
            float4* mo = reinterpret_cast<float4*>(sg.m + ch.begin);
            float4* ve = reinterpret_cast<float4*>(sg.v + ch.begin);
            const uint2* gr = reinterpret_cast<const uint2*>(static_cast<const __nv_bfloat16*>(sg.grad) + ch.begin);
            uint2* wo = reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(sg.wout) + ch.begin);
            const int64_t n4 = ch.len / 4;
            // one group of 4 per thread-iteration: occupancy (not per-thread ILP) hides the
            // fp64 divide/sqrt latency without spilling
            for (int64_t i = threadIdx.x; i < n4; i += blockDim.x) {
                const uint2 g0 = __ldcs(gr + i);
                float4 m0 = __ldcs(ms + i), a0 = __ldcs(mo + i), v0 = __ldcs(ve + i);
                uint2 w0;
                adamw_group4(m0, a0, v0, g0, c, sg.scale, clip, w0);
                __stcs(ms + i, m0);
                __stcs(mo + i, a0);
                __stcs(ve + i, v0);
                __stcs(wo + i, w0);
            }
        } else {
            for (int64_t i = threadIdx.x; i < ch.len; i += blockDim.x) {
                const int64_t e = ch.begin + i;
                float g = load_grad(sg.grad, a.grad_dtype, e);
                if (sg.scale != 1.f) g = __fmul_rn(g, sg.scale);
                if (clip != 1.0) g = (float)__dmul_rn((double)g, clip);
                float ms = sg.master[e], mv = sg.m[e], vv = sg.v[e], wf;
                adamw_elem(ms, mv, vv, g, c, wf);
                sg.master[e] = ms;
                sg.m[e] = mv;
                sg.v[e] = vv;
                if (a.weight_dtype == F32) {
                    static_cast<float*>(sg.wout)[e] =
                        a.round_bf16 ? __uint_as_float((uint32_t)bf16_bits_rne(wf) << 16) : wf;
                } else {
                    static_cast<uint16_t*>(sg.wout)[e] = bf16_bits_rne(wf);
                }
            }
        }
    }
}

__global__ void nonfinite_scan_kernel(const void* __restrict__ g, int dtype, int64_t n, int32_t* flag) {
    bool bad = false;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        bad |= !isfinite(load_grad(g, dtype, i));
    flag_nonfinite(bad, flag);
}

void launch_sumsq_chunks(const OptSeg* segs, const OptChunk* chunks, const int32_t* ids, int nids, int grad_dtype,
                         double* partials, int32_t* nonfinite, cudaStream_t st) {
    if (nids <= 0) return;
    launch_k(sumsq_chunks_kernel, dim3(nids), dim3(256), 0, st, segs, chunks, ids, grad_dtype, partials, nonfinite);
    B2_LAUNCH_CHECK();
}

void launch_norm_final(const double* partials, int n, double* norm_sq, cudaStream_t st) {
    launch_k(norm_final_kernel, dim3(1), dim3(1024), 0, st, partials, n, norm_sq);
    B2_LAUNCH_CHECK();
}

void launch_adamw_chunks(const OptSeg* segs, const OptChunk* chunks, const int32_t* ids, int nids,
                         const OptStepArgs& a, const double* norm_sq, cudaStream_t st,
                         int sm_reserve) {
    if (nids <= 0) return;
    AdamWDev c;
    c.lr = a.lr;
    c.b1 = a.beta1;
    c.b2 = a.beta2;
    c.omb1 = 1.0 - a.beta1;
    c.omb2 = 1.0 - a.beta2;
    c.eps = a.eps;
    c.lr_wd = a.lr * a.weight_decay;
    c.bc1 = a.bc1;
    c.bc2 = a.bc2;
    c.rbc1 = 1.0 / a.bc1;
    c.rbc2 = 1.0 / a.bc2;
    c.lr_rbc1 = a.lr * c.rbc1;
    static int grid_cap = 0, per_sm_blocks = 1;  // resident blocks (persistent grid)
    if (grid_cap == 0) {
        int dev = 0, sms = 148, per_sm = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        B2_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, adamw_chunks_kernel<4>, 256, 0));
        per_sm_blocks = std::max(1, per_sm);
        grid_cap = sms * per_sm_blocks;
    }
    const int grid = std::max(1, std::min(nids, grid_cap - std::max(0, sm_reserve) * per_sm_blocks));
    launch_k(adamw_chunks_kernel<4>, dim3(grid), dim3(256), 0, st, segs, chunks, ids, nids, c, a, norm_sq);
    B2_LAUNCH_CHECK();
}

void launch_nonfinite_scan(const void* g, int dtype, int64_t n, int32_t* flag, cudaStream_t st) {
    if (n <= 0) return;
    nonfinite_scan_kernel<<<adamw_grid(n), 256, 0, st>>>(g, dtype, n, flag);
    B2_LAUNCH_CHECK();
}

}  // namespace b2
