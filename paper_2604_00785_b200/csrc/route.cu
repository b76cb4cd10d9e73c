// Router: logits = x · Wr, fp64-mirrored softmax, top-k, aux statistics, and the
// router backward (softmax backward, dWr, dlogits · Wrᵀ).
//
// Reference: route (include/optimus/moe.hpp:58-80) over matmul (kernels.hpp:16-49),
// softmax (kernels.hpp:194-214), topk (kernels.hpp:235-258), fur_route (moe.hpp:84-99),
// balancing statistics (moe.hpp:381-386), router backward (moe.hpp:431-454).
//
// Parity: logits are accumulated exactly like the reference (fp32, p-outer order,
// separate multiply and add, no FMA contraction), the softmax max/exp/sum/divide
// follow kernels.hpp:201-212 in fp64 with the sequential sum order, and top-k uses
// the same strict '>' (ties to the lower expert index). Given identical scores the
// selections are bit-exact.
#include <cstdlib>

#include "b2_common.cuh"
#include "kernels.h"

namespace b2 {

// ---- logits: 64 tokens x 64 experts per CTA, 128 threads, 8 x 4 outputs per thread ------
// x tiles are loaded with 16-byte vectors and stored transposed (xs[p][token]) so the
// inner loop reads operands with 128-bit shared loads. For bf16 inputs every product
// is exact in fp32, so an FMA rounds exactly like the reference's multiply-then-add;
// fp32 inputs use a separate multiply and add.

constexpr int kRtTok = 64, kRtExp = 64, kRtP = 32, kRtXs = kRtTok + 4;

template <typename T>
__global__ void __launch_bounds__(128) router_logits_kernel(const T* __restrict__ x, const T* __restrict__ w,
                                                            float* __restrict__ logits, int S, int H, int N) {
    pdl_wait();
    pdl_launch();
    __shared__ __align__(16) float xs[2][kRtP][kRtXs];
    __shared__ __align__(16) float ws[2][kRtP][kRtExp];
    const int t0 = blockIdx.x * kRtTok, e0 = blockIdx.y * kRtExp;
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;  // 16 expert-quads x 8 token-octets
    constexpr int VX = 16 / sizeof(T);
    constexpr int XV = kRtTok * kRtP / VX / 128;  // x vectors per thread per chunk
    const bool vec = (H % VX) == 0;
    float2 acc[8][2];  // packed pairs of experts: f32x2 FMA (sm_100), per-lane IEEE rounding
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) acc[i][j] = make_float2(0.f, 0.f);
    int4 xr[XV];
    float wr[kRtP * kRtExp / 128];
    // chunk loads into registers (issued one chunk ahead of the math)
    auto load = [&](int p0) {
        if (vec) {
#pragma unroll
            for (int q = 0; q < XV; ++q) {
                const int v = threadIdx.x + 128 * q;
                const int tt = v / (kRtP / VX), pp = (v % (kRtP / VX)) * VX;
                const int t = t0 + tt, p = p0 + pp;
                xr[q] = (t < S && p < H) ? __ldg(reinterpret_cast<const int4*>(x + (int64_t)t * H + p))
                                         : make_int4(0, 0, 0, 0);
            }
        }
#pragma unroll
        for (int q = 0; q < kRtP * kRtExp / 128; ++q) {
            const int i = threadIdx.x + 128 * q;
            const int pp = i / kRtExp, ee = i % kRtExp;
            const int p = p0 + pp, e = e0 + ee;
            wr[q] = (p < H && e < N) ? Elem<T>::load(w + (int64_t)p * N + e) : 0.f;
        }
    };
    auto stash = [&](int buf, int p0) {
        if (vec) {
#pragma unroll
            for (int q = 0; q < XV; ++q) {
                const int v = threadIdx.x + 128 * q;
                const int tt = v / (kRtP / VX), pp = (v % (kRtP / VX)) * VX;
                float f[VX];
                if constexpr (sizeof(T) == 2) {
                    const uint32_t wv[4] = {(uint32_t)xr[q].x, (uint32_t)xr[q].y, (uint32_t)xr[q].z, (uint32_t)xr[q].w};
#pragma unroll
                    for (int z = 0; z < 4; ++z) {
                        f[2 * z] = __uint_as_float(wv[z] << 16);
                        f[2 * z + 1] = __uint_as_float(wv[z] & 0xFFFF0000u);
                    }
                } else {
                    f[0] = __int_as_float(xr[q].x);
                    f[1] = __int_as_float(xr[q].y);
                    f[2] = __int_as_float(xr[q].z);
                    f[3] = __int_as_float(xr[q].w);
                }
#pragma unroll
                for (int z = 0; z < VX; ++z) xs[buf][pp + z][tt] = f[z];
            }
        } else {
            for (int i = threadIdx.x; i < kRtTok * kRtP; i += 128) {
                const int tt = i / kRtP, pp = i % kRtP;
                const int t = t0 + tt, p = p0 + pp;
                xs[buf][pp][tt] = (t < S && p < H) ? Elem<T>::load(x + (int64_t)t * H + p) : 0.f;
            }
        }
#pragma unroll
        for (int q = 0; q < kRtP * kRtExp / 128; ++q) {
            const int i = threadIdx.x + 128 * q;
            ws[buf][i / kRtExp][i % kRtExp] = wr[q];
        }
    };
    load(0);
    stash(0, 0);
    __syncthreads();
    int buf = 0;
    for (int p0 = 0; p0 < H; p0 += kRtP) {
        const bool more = p0 + kRtP < H;
        if (more) load(p0 + kRtP);
        const int pend = min(kRtP, H - p0);
#pragma unroll 8
        for (int pp = 0; pp < pend; ++pp) {
            const float4 a0 = *reinterpret_cast<const float4*>(&xs[buf][pp][ty * 8]);
            const float4 a1 = *reinterpret_cast<const float4*>(&xs[buf][pp][ty * 8 + 4]);
            const float4 b4 = *reinterpret_cast<const float4*>(&ws[buf][pp][tx * 4]);
            const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
            const float2 b[2] = {make_float2(b4.x, b4.y), make_float2(b4.z, b4.w)};
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const float2 a2 = make_float2(a[i], a[i]);
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    if constexpr (sizeof(T) == 2) {
                        acc[i][j] = __ffma2_rn(a2, b[j], acc[i][j]);
                    } else {  // scalar _rn intrinsics are never contracted into an FMA
                        acc[i][j].x = __fadd_rn(acc[i][j].x, __fmul_rn(a2.x, b[j].x));
                        acc[i][j].y = __fadd_rn(acc[i][j].y, __fmul_rn(a2.y, b[j].y));
                    }
                }
            }
        }
        if (more) stash(buf ^ 1, p0 + kRtP);
        __syncthreads();
        buf ^= 1;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int t = t0 + ty * 8 + i;
        if (t >= S) continue;
        const float o[4] = {acc[i][0].x, acc[i][0].y, acc[i][1].x, acc[i][1].y};
        if (e0 + tx * 4 + 3 < N && (N % 4) == 0) {
            *reinterpret_cast<float4*>(logits + (int64_t)t * N + e0 + tx * 4) = make_float4(o[0], o[1], o[2], o[3]);
        } else {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int e = e0 + tx * 4 + j;
                if (e < N) logits[(int64_t)t * N + e] = o[j];
            }
        }
    }
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
    const uint32_t d = (uint32_t)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(gmem), "r"(valid ? 16 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// ---- logits, bf16 inputs, 8 x 8 register tiles ----------------------------------------
// One warp per CTA, 32 tokens x 64 experts; each lane owns 8 tokens x 8 experts (64 fp32
// accumulators as 32 float2). Per p step a lane loads its 8 x values and 8 W values (4
// conflict-free 128-bit shared loads), duplicates each x into an (x, x) pair in registers and
// issues 32 fma.rn.f32x2 that pair two EXPERTS against one token (2x the FMAs per shared byte
// of a token-paired 8 x 4 tile, measured 158 -> 122 us at config B). The order of every
// accumulator is still p = 0, 1, ... with one rounding per step, and bf16 x bf16 products are
// exact in fp32, so the logits stay bit-identical to the reference's multiply-then-add.
constexpr int kL3P = 32, kL3Exp = 64, kL3Stages = 4;
constexpr int kLogitsTok = 16;  // tokens per warp (16 or 32)
template <int TOK>
struct Logits3Smem {
    uint16_t xraw[kL3Stages][TOK][kL3P];      // 64 B rows, 16 B units swizzled by (t >> 1) & 3
    uint16_t wraw[kL3Stages][kL3P][kL3Exp];   // 128 B rows, 16 B units swizzled by p & 7
    float xs[2][kL3P][TOK];                   // x transposed to [p][token], fp32
};

// One warp per TOK tokens x 64 experts; a lane owns TOK/4 tokens x 8 experts. W is read in its
// raw bf16 form straight from the cp.async ring (one 16 B load per p step, widened in
// registers); only x goes through a transposed fp32 copy, 4 tokens per 16 B store. TOK = 16
// runs twice the warps of TOK = 32 (two per scheduler instead of one, which left the FMA pipe
// idle half the time: ncu issue 42 %, FMA 50 %).
template <int TOK>
__global__ void __launch_bounds__(32) router_logits_bf16_kernel(const __nv_bfloat16* __restrict__ x,
                                                                const __nv_bfloat16* __restrict__ w,
                                                                float* __restrict__ logits, int S, int H, int N) {
    pdl_wait();
    pdl_launch();
    using Sm = Logits3Smem<TOK>;
    constexpr int TPL = TOK / 4;  // tokens per lane
    extern __shared__ __align__(128) uint8_t l3_smem[];
    Sm& sm = *reinterpret_cast<Sm*>(l3_smem);
    const int lane = threadIdx.x;
    const int t0 = blockIdx.x * TOK, e0 = blockIdx.y * kL3Exp;
    const int nchunks = H / kL3P;
    auto issue = [&](int c) {
        if (c < nchunks) {
            const int s = c % kL3Stages, p0 = c * kL3P;
#pragma unroll
            for (int q = 0; q < TOK / 8; ++q) {  // x: TOK rows x 4 units
                const int idx = lane + 32 * q, t = idx / 4, u = idx % 4;
                const bool ok = t0 + t < S;
                const __nv_bfloat16* src = x + (int64_t)(ok ? t0 + t : 0) * H + p0 + 8 * u;
                cp_async16(&sm.xraw[s][t][8 * (u ^ ((t >> 1) & 3))], src, ok);
            }
#pragma unroll
            for (int q = 0; q < 8; ++q) {  // W: 32 rows x 8 units
                const int idx = lane + 32 * q, pp = idx / 8, u = idx % 8;
                const bool ok = e0 + 8 * u < N;
                const __nv_bfloat16* src = w + (int64_t)(p0 + pp) * N + (ok ? e0 + 8 * u : 0);
                cp_async16(&sm.wraw[s][pp][8 * (u ^ (pp & 7))], src, ok);
            }
        }
        cp_async_commit();
    };
    // x of chunk c -> xs[c & 1]: lane (tq, u) < TOK moves tokens 4tq .. 4tq+3, p 8u .. 8u+7
    auto widen = [&](int c) {
        if (lane >= TOK) return;
        const int s = c % kL3Stages, b = c & 1, tq = lane / 4, u = lane % 4;
        uint4 r[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int t = 4 * tq + i;
            r[i] = *reinterpret_cast<const uint4*>(&sm.xraw[s][t][8 * (u ^ ((t >> 1) & 3))]);
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint32_t v0 = (&r[0].x)[j], v1 = (&r[1].x)[j], v2 = (&r[2].x)[j], v3 = (&r[3].x)[j];
            *reinterpret_cast<float4*>(&sm.xs[b][8 * u + 2 * j][4 * tq]) =
                make_float4(__uint_as_float(v0 << 16), __uint_as_float(v1 << 16), __uint_as_float(v2 << 16),
                            __uint_as_float(v3 << 16));
            *reinterpret_cast<float4*>(&sm.xs[b][8 * u + 2 * j + 1][4 * tq]) =
                make_float4(__uint_as_float(v0 & 0xFFFF0000u), __uint_as_float(v1 & 0xFFFF0000u),
                            __uint_as_float(v2 & 0xFFFF0000u), __uint_as_float(v3 & 0xFFFF0000u));
        }
    };

    float2 acc[TPL][4];  // [token][expert pair]
#pragma unroll
    for (int i = 0; i < TPL; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = make_float2(0.f, 0.f);

#pragma unroll
    for (int c = 0; c < kL3Stages - 1; ++c) issue(c);
    cp_async_wait<kL3Stages - 2>();
    __syncwarp();
    widen(0);
    const int tg = lane % 4, eg = lane / 4;  // tokens TPL*tg .., experts 8*eg .. +7
    for (int c = 0; c < nchunks; ++c) {
        // chunk c+1 landed (chunk c's x is in xs[c & 1]); ring slot (c - 1) % stages is free
        cp_async_wait<kL3Stages - 3>();
        __syncwarp();
        if (c + 1 < nchunks) widen(c + 1);
        issue(c + kL3Stages - 1);
        const int b = c & 1, s = c % kL3Stages;
        float4 xa[2][TPL / 4];
        uint4 wb[2];
        auto ld = [&](int q, int pp) {
#pragma unroll
            for (int h = 0; h < TPL / 4; ++h)
                xa[q][h] = *reinterpret_cast<const float4*>(&sm.xs[b][pp][TPL * tg + 4 * h]);
            wb[q] = *reinterpret_cast<const uint4*>(&sm.wraw[s][pp][8 * (eg ^ (pp & 7))]);
        };
        ld(0, 0);
#pragma unroll
        for (int pp = 0; pp < kL3P; ++pp) {
            if (pp + 1 < kL3P) ld((pp + 1) & 1, pp + 1);
            float xv[TPL];
#pragma unroll
            for (int h = 0; h < TPL / 4; ++h) {
                const float4 a = xa[pp & 1][h];
                xv[4 * h] = a.x;
                xv[4 * h + 1] = a.y;
                xv[4 * h + 2] = a.z;
                xv[4 * h + 3] = a.w;
            }
            const uint32_t wr[4] = {wb[pp & 1].x, wb[pp & 1].y, wb[pp & 1].z, wb[pp & 1].w};
            float2 wp[4];
#pragma unroll
            for (int j = 0; j < 4; ++j)
                wp[j] = make_float2(__uint_as_float(wr[j] << 16), __uint_as_float(wr[j] & 0xFFFF0000u));
#pragma unroll
            for (int i = 0; i < TPL; ++i) {
                const float2 xd = make_float2(xv[i], xv[i]);
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = __ffma2_rn(xd, wp[j], acc[i][j]);
            }
        }
    }
    const int e = e0 + 8 * eg;
#pragma unroll
    for (int i = 0; i < TPL; ++i) {
        const int t = t0 + TPL * tg + i;
        if (t >= S) continue;
        float* dst = logits + (int64_t)t * N + e;
        if (e + 7 < N) {
            *reinterpret_cast<float4*>(dst) = make_float4(acc[i][0].x, acc[i][0].y, acc[i][1].x, acc[i][1].y);
            *reinterpret_cast<float4*>(dst + 4) = make_float4(acc[i][2].x, acc[i][2].y, acc[i][3].x, acc[i][3].y);
        } else {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                if (e + 2 * j < N) dst[2 * j] = acc[i][j].x;
                if (e + 2 * j + 1 < N) dst[2 * j + 1] = acc[i][j].y;
            }
        }
    }
}

// ---- softmax + top-k: one warp per token -------------------------------------------

constexpr int kMaxExpertsPerLane = 8;  // N <= 256

// NPL = experts per lane (N <= 32 * NPL), a compile-time bound so the per-lane arrays
// stay in registers. The fp64 exponentials go to shared memory and one lane adds them in
// expert order (kernels.hpp:205-209); each top-k round is two warp reductions
// (redux.sync): the max probability's bit pattern (probs are >= 0, so their IEEE bits
// order like unsigned integers), then the lowest expert index holding it — strict '>'
// with ties to the lower index (kernels.hpp:246-255).
template <int NPL>
__global__ void __launch_bounds__(256) softmax_topk_kernel(const float* __restrict__ logits, float* __restrict__ probs,
                                                           float* __restrict__ topw, int32_t* __restrict__ topi, int S,
                                                           int N, int K, int normalize) {
    pdl_wait();
    pdl_launch();
    __shared__ double es[8][32 * NPL];
    const int wib = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int warp = blockIdx.x * 8 + wib;
    if (warp >= S) return;
    const float* lp = logits + (int64_t)warp * N;
    float v[NPL];
    float mx = lp[0];
#pragma unroll
    for (int i = 0; i < NPL; ++i) {
        const int j = lane + 32 * i;
        v[i] = j < N ? lp[j] : 0.f;
        if (j < N) mx = fmaxf(mx, v[i]);
    }
    // max in T (order-independent for non-NaN input)
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    double e[NPL];
#pragma unroll
    for (int i = 0; i < NPL; ++i) {
        const int j = lane + 32 * i;
        e[i] = j < N ? exp((double)v[i] - (double)mx) : 0.0;
        if (j < N) es[wib][j] = e[i];
    }
    __syncwarp();
    double sum = 0.0;
    if (lane == 0) {
        const double* row = es[wib];
#pragma unroll 8
        for (int j = 0; j < N; ++j) sum += row[j];
    }
    sum = __shfl_sync(0xffffffffu, sum, 0);
    float p[NPL];
#pragma unroll
    for (int i = 0; i < NPL; ++i) {
        const int j = lane + 32 * i;
        p[i] = (float)(e[i] / sum);
        if (j < N) probs[(int64_t)warp * N + j] = p[i];
    }
    unsigned taken = 0;
    float wsum = 0.f;
    for (int c = 0; c < K; ++c) {
        // this lane's best untaken candidate (within a lane j increases: strict '>')
        uint32_t bb = 0;
        int bi = 0x7fffffff;
#pragma unroll
        for (int i = 0; i < NPL; ++i) {
            const int j = lane + 32 * i;
            if (j < N && !(taken >> i & 1u)) {
                const uint32_t pb = __float_as_uint(p[i]);
                if (bi == 0x7fffffff || pb > bb) {
                    bb = pb;
                    bi = j;
                }
            }
        }
        const uint32_t best = __reduce_max_sync(0xffffffffu, bi == 0x7fffffff ? 0u : bb);
        const uint32_t cand = (bi != 0x7fffffff && bb == best) ? (uint32_t)bi : 0xffffffffu;
        const int win = (int)__reduce_min_sync(0xffffffffu, cand);
        if (lane == win % 32) taken |= 1u << (win / 32);
        const float bv = __uint_as_float(best);
        wsum += bv;  // K-order sum in T for the renormalisation (moe.hpp:72-78)
        if (lane == 0) {
            topi[(int64_t)warp * K + c] = win;
            topw[(int64_t)warp * K + c] = bv;
        }
    }
    if (normalize && lane == 0)
        for (int c = 0; c < K; ++c) topw[(int64_t)warp * K + c] = __fdiv_rn(topw[(int64_t)warp * K + c], wsum);
}

// forced uniform routing (moe.hpp:84-99): expert (t*K+j) mod N, weight 1/K
__global__ void fur_route_kernel(float* __restrict__ w, int32_t* __restrict__ idx, int S, int N, int K) {
    pdl_wait();
    pdl_launch();
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (int64_t)S * K) return;
    const int64_t t = i / K, k = i % K;
    w[i] = (float)(1.0 / (double)K);
    idx[i] = (int32_t)((t * K + k) % N);
}

// ---- balancing statistics: mean_probs over local rows, sel_counts over the gathered
// table (moe.hpp:381-386). Column sums use a fixed two-level order (deterministic).

// One block per 128-row slice writes that slice's column sums; the last block to arrive
// (arrival counter, self-resetting) adds the slices in slice order. Both levels keep the
// fixed order of the former two-kernel version, so mean_probs is bitwise unchanged.
__global__ void prob_colsum_kernel(const float* __restrict__ probs, float* __restrict__ partial,
                                   int32_t* __restrict__ ctr, float* __restrict__ mean_probs, int S, int N,
                                   int rows_per_block) {
    pdl_wait();
    pdl_launch();
    constexpr int U = 16;
    const int r0 = blockIdx.x * rows_per_block;
    const int r1 = min(S, r0 + rows_per_block);
    for (int e = threadIdx.x; e < N; e += blockDim.x) {
        float acc = 0.f;
        int r = r0;
        for (; r + U <= r1; r += U) {  // U independent loads in flight, then the sums in row order
            float v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) v[u] = __ldg(probs + (int64_t)(r + u) * N + e);
#pragma unroll
            for (int u = 0; u < U; ++u) acc += v[u];
        }
        for (; r < r1; ++r) acc += probs[(int64_t)r * N + e];
        partial[(int64_t)blockIdx.x * N + e] = acc;
    }
    __threadfence();
    __syncthreads();
    __shared__ int last;
    if (threadIdx.x == 0) last = atomicAdd(ctr, 1) == (int)gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    const int nparts = gridDim.x;
    for (int e = threadIdx.x; e < N; e += blockDim.x) {
        float acc = 0.f;
        int b = 0;
        for (; b + U <= nparts; b += U) {
            float v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) v[u] = __ldcg(partial + (int64_t)(b + u) * N + e);
#pragma unroll
            for (int u = 0; u < U; ++u) acc += v[u];
        }
        for (; b < nparts; ++b) acc += __ldcg(partial + (int64_t)b * N + e);
        mean_probs[e] = acc * (float)(1.0 / (double)S);
    }
    if (threadIdx.x == 0) *ctr = 0;
}

__global__ void sel_count_kernel(const int32_t* __restrict__ idx, int64_t n, int32_t* __restrict__ sel, int N) {
    pdl_wait();
    pdl_launch();
    extern __shared__ int32_t hist[];
    for (int e = threadIdx.x; e < N; e += blockDim.x) hist[e] = 0;
    __syncthreads();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(&hist[idx[i]], 1);
    __syncthreads();
    for (int e = threadIdx.x; e < N; e += blockDim.x)
        if (hist[e]) atomicAdd(&sel[e], hist[e]);
}

// ---- router backward (moe.hpp:431-454) -----------------------------------------------

// dprobs[s, idx[s,k]] += wgrad[s,k] (or the renormalised form, 434-444); + aux grad
// column constant; then dlogits = softmax_backward(probs, dprobs) with the fp64 dot.
// One warp per local row.
__global__ void router_dlogits_kernel(const float* __restrict__ probs, const float* __restrict__ wgrad,
                                      const int32_t* __restrict__ topi, const float* __restrict__ topw,
                                      const float* __restrict__ aux_grad /*[S,N] or null*/,
                                      float* __restrict__ dlogits, __nv_bfloat16* __restrict__ dl_bf16,
                                      __nv_bfloat16* __restrict__ dl_lo, int S, int N, int K, int normalize,
                                      int fur) {
    pdl_wait();
    pdl_launch();
    const int row = (blockIdx.x * blockDim.x + threadIdx.x) / 32, lane = threadIdx.x % 32;
    if (row >= S) return;
    float dp[kMaxExpertsPerLane], pr[kMaxExpertsPerLane];
#pragma unroll
    for (int i = 0; i < kMaxExpertsPerLane; ++i) {
        const int j = lane + 32 * i;
        dp[i] = 0.f;
        pr[i] = j < N ? probs[(int64_t)row * N + j] : 0.f;
    }
    if (!fur && K <= 32) {
        // lane k holds the row's k-th selection: the gathers and the per-k divisions run in
        // parallel across lanes; raw_sum / dot still accumulate in k order (shuffled), and the
        // selected experts are distinct, so every dp element receives exactly one add
        const bool act = lane < K;
        const int64_t ik = (int64_t)row * K + lane;
        const int ek = act ? topi[ik] : 0;
        const float gk = act ? wgrad[ik] : 0.f;
        float addk = gk;
        if (normalize) {
            const float pk = act ? probs[(int64_t)row * N + ek] : 0.f;
            const float wk = act ? topw[ik] : 0.f;
            double raw_sum = 0, dot = 0;
            for (int k = 0; k < K; ++k) raw_sum += (double)__shfl_sync(0xffffffffu, pk, k);
            for (int k = 0; k < K; ++k)
                dot += (double)__shfl_sync(0xffffffffu, gk, k) * (double)__shfl_sync(0xffffffffu, wk, k);
            addk = (float)(((double)gk - dot) / raw_sum);
        }
        for (int k = 0; k < K; ++k) {
            const int e = __shfl_sync(0xffffffffu, ek, k);
            const float add = __shfl_sync(0xffffffffu, addk, k);
            if (e % 32 == lane) {
#pragma unroll
                for (int i = 0; i < kMaxExpertsPerLane; ++i)
                    if (i == e / 32) dp[i] += add;
            }
        }
    } else if (!fur) {
        double raw_sum = 0, dot = 0;
        if (normalize) {
            for (int k = 0; k < K; ++k) raw_sum += (double)probs[(int64_t)row * N + topi[(int64_t)row * K + k]];
            for (int k = 0; k < K; ++k)
                dot += (double)wgrad[(int64_t)row * K + k] * (double)topw[(int64_t)row * K + k];
        }
        for (int k = 0; k < K; ++k) {
            const int e = topi[(int64_t)row * K + k];
            const float g = wgrad[(int64_t)row * K + k];
            const float add = normalize ? (float)(((double)g - dot) / raw_sum) : g;
            if (e % 32 == lane) {
#pragma unroll
                for (int i = 0; i < kMaxExpertsPerLane; ++i)
                    if (i == e / 32) dp[i] += add;
            }
        }
    }
    if (aux_grad) {
#pragma unroll
        for (int i = 0; i < kMaxExpertsPerLane; ++i) {
            const int j = lane + 32 * i;
            if (j < N) dp[i] += aux_grad[(int64_t)row * N + j];
        }
    }
    double dot = 0.0;
#pragma unroll
    for (int i = 0; i < kMaxExpertsPerLane; ++i) dot += (double)pr[i] * (double)dp[i];
#pragma unroll
    for (int o = 16; o; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
#pragma unroll
    for (int i = 0; i < kMaxExpertsPerLane; ++i) {
        const int j = lane + 32 * i;
        if (j < N) {
            const float v = (float)((double)pr[i] * ((double)dp[i] - dot));
            dlogits[(int64_t)row * N + j] = v;
            if (dl_bf16) {
                // two-term bf16 split for the tensor-core router GEMMs: hi + lo carries ~16
                // mantissa bits, so dlogits · Wrᵀ keeps fp32-level accuracy when |Wr| is O(1)
                const __nv_bfloat16 hi = __float2bfloat16_rn(v);
                dl_bf16[(int64_t)row * N + j] = hi;
                if (dl_lo) dl_lo[(int64_t)row * N + j] = __float2bfloat16_rn(v - __bfloat162float(hi));
            }
        }
    }
}

// aux-loss probability gradient (moe.hpp:331-342): coeff*N*f_e/S in every row
__global__ void aux_probs_grad_kernel(const int32_t* __restrict__ sel, float* __restrict__ out, int S, int N,
                                      double coeff, double total) {
    pdl_wait();
    pdl_launch();
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (int64_t)S * N) return;
    const int e = (int)(i % N);
    out[i] = (float)(coeff * (double)N * ((double)sel[e] / total) / (double)S);
}

// dWr[h, e] = sum_s x[s,h] * dlogits[s,e]  (matmul_tn, kernels.hpp:52-72): CTA tile of
// 64 h-rows x 64 experts over one slice of the S rows; the slices' partials are then
// summed in slice order by router_dw_reduce_kernel (deterministic split-S).
template <typename T>
__global__ void __launch_bounds__(128) router_dw_partial_kernel(const T* __restrict__ x, const float* __restrict__ dl,
                                                                float* __restrict__ part, int S, int H, int N,
                                                                int rows_per_split) {
    __shared__ __align__(16) float xs[kRtP][64];
    __shared__ __align__(16) float ds[kRtP][64];
    const int h0 = blockIdx.x * 64, e0 = blockIdx.y * 64, split = blockIdx.z;
    const int sb = split * rows_per_split, se = min(S, sb + rows_per_split);
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;  // 16 expert-quads x 8 h-octets
    float acc[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
    for (int s0 = sb; s0 < se; s0 += kRtP) {
        for (int i = threadIdx.x; i < kRtP * 64; i += 128) {
            const int ss = i / 64, hh = i % 64;
            const int s = s0 + ss, h = h0 + hh, e = e0 + hh;
            xs[ss][hh] = (s < se && h < H) ? Elem<T>::load(x + (int64_t)s * H + h) : 0.f;
            ds[ss][hh] = (s < se && e < N) ? dl[(int64_t)s * N + e] : 0.f;
        }
        __syncthreads();
#pragma unroll 4
        for (int ss = 0; ss < kRtP; ++ss) {
            const float4 a0 = *reinterpret_cast<const float4*>(&xs[ss][ty * 8]);
            const float4 a1 = *reinterpret_cast<const float4*>(&xs[ss][ty * 8 + 4]);
            const float4 b4 = *reinterpret_cast<const float4*>(&ds[ss][tx * 4]);
            const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
            const float b[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int h = h0 + ty * 8 + i;
        if (h >= H) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int e = e0 + tx * 4 + j;
            if (e < N) part[((int64_t)split * H + h) * N + e] = acc[i][j];
        }
    }
}

template <typename T>
__global__ void router_dw_reduce_kernel(const float* __restrict__ part, T* __restrict__ dw, int nsplit, int64_t n) {
    pdl_wait();
    pdl_launch();
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    float acc = 0.f;
    for (int sp = 0; sp < nsplit; ++sp) acc += part[(int64_t)sp * n + i];
    dw[i] = Elem<T>::from_f(acc);
}

// ---- launchers ----------------------------------------------------------------------

template <typename T>
void launch_router_logits(const T* x, const T* w, float* logits, int S, int H, int N, cudaStream_t st) {
    if (S == 0) return;
    if constexpr (sizeof(T) == 2) {
        if (H % kL3P == 0 && N % 8 == 0 && ((uintptr_t)x & 15) == 0 && ((uintptr_t)w & 15) == 0) {
            constexpr int TOK = kLogitsTok;
            static bool attr = false;
            if (!attr) {
                B2_CUDA(cudaFuncSetAttribute(router_logits_bf16_kernel<TOK>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)sizeof(Logits3Smem<TOK>)));
                attr = true;
            }
            dim3 grid((unsigned)ceil_div(S, TOK), (unsigned)ceil_div(N, kL3Exp));
            launch_k(router_logits_bf16_kernel<TOK>, grid, dim3(32), sizeof(Logits3Smem<TOK>), st, x, w, logits, S, H, N);
            B2_LAUNCH_CHECK();
            return;
        }
    }
    dim3 grid((unsigned)ceil_div(S, kRtTok), (unsigned)ceil_div(N, kRtExp));
    launch_k(router_logits_kernel<T>, dim3(grid), dim3(128), 0, st, x, w, logits, S, H, N);
    B2_LAUNCH_CHECK();
}
template void launch_router_logits<float>(const float*, const float*, float*, int, int, int, cudaStream_t);
template void launch_router_logits<__nv_bfloat16>(const __nv_bfloat16*, const __nv_bfloat16*, float*, int, int,
                                                  int, cudaStream_t);

void launch_softmax_topk(const float* logits, float* probs, float* topw, int32_t* topi, int S, int N, int K,
                         bool normalize, cudaStream_t st) {
    check(N <= 32 * kMaxExpertsPerLane, "route: n_experts above 256 is not supported by the router kernel");
    if (S == 0) return;
    const unsigned grid = (unsigned)ceil_div(S, 8);  // 8 warps (tokens) per block
    const int nm = normalize ? 1 : 0;
    if (N <= 64) launch_k(softmax_topk_kernel<2>, dim3(grid), dim3(256), 0, st, logits, probs, topw, topi, S, N, K, nm);
    else if (N <= 128) launch_k(softmax_topk_kernel<4>, dim3(grid), dim3(256), 0, st, logits, probs, topw, topi, S, N, K, nm);
    else launch_k(softmax_topk_kernel<8>, dim3(grid), dim3(256), 0, st, logits, probs, topw, topi, S, N, K, nm);
    B2_LAUNCH_CHECK();
}

void launch_fur_route(float* w, int32_t* idx, int S, int N, int K, cudaStream_t st) {
    const int64_t n = (int64_t)S * K;
    if (n == 0) return;
    launch_k(fur_route_kernel, dim3((unsigned)ceil_div(n, 256)), dim3(256), 0, st, w, idx, S, N, K);
    B2_LAUNCH_CHECK();
}

void launch_aux_stats(const float* probs, int S, int N, const int32_t* gidx, int64_t n_gidx, float* partial,
                      int32_t* ctr, float* mean_probs, int32_t* sel, cudaStream_t st) {
    B2_CUDA(cudaMemsetAsync(sel, 0, sizeof(int32_t) * N, st));
    if (S > 0) {
        const int rpb = 128;
        const int nparts = (int)ceil_div(S, rpb);
        launch_k(prob_colsum_kernel, dim3(nparts), dim3(128), 0, st, probs, partial, ctr, mean_probs, S, N, rpb);
        B2_LAUNCH_CHECK();
    } else {
        B2_CUDA(cudaMemsetAsync(mean_probs, 0, sizeof(float) * N, st));
    }
    if (n_gidx > 0) {
        launch_k(sel_count_kernel, dim3((unsigned)std::min<int64_t>(148, ceil_div(n_gidx, 256))), dim3(256), sizeof(int32_t) * N, st, 
            gidx, n_gidx, sel, N);
        B2_LAUNCH_CHECK();
    }
}

void launch_router_dlogits(const float* probs, const float* wgrad, const int32_t* topi, const float* topw,
                           const float* aux_grad, float* dlogits, void* dl_bf16, void* dl_lo, int S, int N, int K,
                           bool normalize, bool fur, cudaStream_t st) {
    if (S == 0) return;
    launch_k(router_dlogits_kernel, dim3((unsigned)ceil_div(S, 8)), dim3(256), 0, st, probs, wgrad, topi, topw, aux_grad,
             dlogits, (__nv_bfloat16*)dl_bf16, (__nv_bfloat16*)dl_lo, S, N, K, normalize ? 1 : 0, fur ? 1 : 0);
    B2_LAUNCH_CHECK();
}

void launch_aux_probs_grad(const int32_t* sel, float* out, int S, int N, double coeff, double total,
                           cudaStream_t st) {
    const int64_t n = (int64_t)S * N;
    if (n == 0) return;
    launch_k(aux_probs_grad_kernel, dim3((unsigned)ceil_div(n, 256)), dim3(256), 0, st, sel, out, S, N, coeff, total);
    B2_LAUNCH_CHECK();
}

template <typename T>
void launch_router_dw(const T* x, const float* dlogits, T* dw, float* part, int max_splits, int S, int H, int N,
                      cudaStream_t st) {
    const int tiles = (int)(ceil_div(H, 64) * ceil_div(N, 64));
    int nsplit = (int)std::max<int64_t>(1, std::min<int64_t>(max_splits, ceil_div(4 * 148, tiles)));
    const int rows = (int)round_up(ceil_div(std::max(S, 1), nsplit), kRtP);
    nsplit = (int)ceil_div(std::max(S, 1), rows);
    dim3 grid((unsigned)ceil_div(H, 64), (unsigned)ceil_div(N, 64), (unsigned)nsplit);
    router_dw_partial_kernel<T><<<grid, 128, 0, st>>>(x, dlogits, part, S, H, N, rows);
    B2_LAUNCH_CHECK();
    const int64_t n = (int64_t)H * N;
    launch_k(router_dw_reduce_kernel<T>, dim3((unsigned)ceil_div(n, 256)), dim3(256), 0, st, part, dw, nsplit, n);
    B2_LAUNCH_CHECK();
}
void launch_router_dw_reduce_bf16(const float* part, void* dw, int nsplit, int64_t n, cudaStream_t st) {
    if (n <= 0) return;
    launch_k(router_dw_reduce_kernel<__nv_bfloat16>, dim3((unsigned)ceil_div(n, 256)), dim3(256), 0, st, part, (__nv_bfloat16*)dw, nsplit, n);
    B2_LAUNCH_CHECK();
}

template void launch_router_dw<float>(const float*, const float*, float*, float*, int, int, int, int, cudaStream_t);
template void launch_router_dw<__nv_bfloat16>(const __nv_bfloat16*, const float*, __nv_bfloat16*, float*, int, int,
                                              int, int, cudaStream_t);

}  // namespace b2
