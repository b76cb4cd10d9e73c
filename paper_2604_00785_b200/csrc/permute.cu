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
#include <type_traits>

#include "b2_common.cuh"
#include "kernels.h"

namespace b2 {

template <typename T>
__device__ __forceinline__ bool vec_ok(int H) {
    return ((int64_t)H * (int64_t)sizeof(T)) % 16 == 0;
}

// 16-byte vectors of T as fp32 lanes
template <typename T>
struct V16 {
    static constexpr int n = 16 / sizeof(T);
    __device__ __forceinline__ static void load(const T* p, float* f) {
        const int4 v = __ldg(reinterpret_cast<const int4*>(p));
        if constexpr (sizeof(T) == 4) {
            f[0] = __int_as_float(v.x); f[1] = __int_as_float(v.y); f[2] = __int_as_float(v.z); f[3] = __int_as_float(v.w);
        } else {
            const uint32_t w[4] = {(uint32_t)v.x, (uint32_t)v.y, (uint32_t)v.z, (uint32_t)v.w};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                f[2 * q] = __uint_as_float(w[q] << 16);
                f[2 * q + 1] = __uint_as_float(w[q] & 0xFFFF0000u);
            }
        }
    }
    __device__ __forceinline__ static void unpack(const int4 v, float* f) {
        if constexpr (sizeof(T) == 4) {
            f[0] = __int_as_float(v.x); f[1] = __int_as_float(v.y); f[2] = __int_as_float(v.z); f[3] = __int_as_float(v.w);
        } else {
            const uint32_t w[4] = {(uint32_t)v.x, (uint32_t)v.y, (uint32_t)v.z, (uint32_t)v.w};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                f[2 * q] = __uint_as_float(w[q] << 16);
                f[2 * q + 1] = __uint_as_float(w[q] & 0xFFFF0000u);
            }
        }
    }
    __device__ __forceinline__ static void store(T* p, const float* f) {
        int4 v;
        if constexpr (sizeof(T) == 4) {
            v = make_int4(__float_as_int(f[0]), __float_as_int(f[1]), __float_as_int(f[2]), __float_as_int(f[3]));
        } else {
            uint32_t w[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                __nv_bfloat162 b = __floats2bfloat162_rn(f[2 * q], f[2 * q + 1]);
                w[q] = *reinterpret_cast<uint32_t*>(&b);
            }
            v = make_int4((int)w[0], (int)w[1], (int)w[2], (int)w[3]);
        }
        *reinterpret_cast<int4*>(p) = v;
    }
};

// mlp_in[prow] = x[prow_src[prow]] (zero row when prow_src < 0); rows < *p_total
template <typename T>
__global__ void gather_rows_kernel(const T* __restrict__ x, const int32_t* __restrict__ prow_src,
                                   const int32_t* __restrict__ p_total, T* __restrict__ out, int H, int64_t pmax) {
    pdl_wait();
    pdl_launch();
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

// The same rows written token-major: warp per token t reads x[t] ONCE (up to 8 x 16 B per lane
// in flight) and writes it to each of its padded rows slot_prow[cec[t] .. cec[t+1]); then the
// pad rows (prow_src < 0, rows < *p_total) are zeroed. The row-major gather above re-reads a
// token's row for each of its K rows, which the streaming writes evict from L2 in between
// (ncu, round 1: 849 MB of DRAM traffic for 604 MB of algorithmic bytes).
template <typename T>
__global__ void gather_tokens_kernel(const T* __restrict__ x, const int32_t* __restrict__ cec,
                                     const int32_t* __restrict__ slot_prow, int T_tok,
                                     const int32_t* __restrict__ prow_src, const int32_t* __restrict__ p_total,
                                     T* __restrict__ out, int H, int64_t pmax) {
    pdl_wait();
    pdl_launch();
    const int lane = threadIdx.x % 32;
    const int64_t warps = (int64_t)gridDim.x * blockDim.x / 32;
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
    const int nv = (int)((int64_t)H * sizeof(T) / 16);  // launcher: rows are 16-byte multiples
    constexpr int B = 8;
    for (int64_t t = w0; t < T_tok; t += warps) {
        const int j0 = cec[t], j1 = cec[t + 1];
        if (j0 == j1) continue;
        const int4* src = reinterpret_cast<const int4*>(x + t * H);
        for (int v0 = 0; v0 < nv; v0 += 32 * B) {
            int4 val[B];
#pragma unroll
            for (int b = 0; b < B; ++b) {
                const int v = v0 + lane + 32 * b;
                if (v < nv) val[b] = __ldg(src + v);
            }
            for (int j = j0; j < j1; ++j) {
                int4* dst = reinterpret_cast<int4*>(out + (int64_t)slot_prow[j] * H);
#pragma unroll
                for (int b = 0; b < B; ++b) {
                    const int v = v0 + lane + 32 * b;
                    if (v < nv) dst[v] = val[b];
                }
            }
        }
    }
    const int64_t P = min((int64_t)*p_total, pmax);
    for (int64_t r = w0; r < P; r += warps) {
        if (prow_src[r] >= 0) continue;
        int4* d4 = reinterpret_cast<int4*>(out + r * H);
        for (int v = lane; v < nv; v += 32) d4[v] = make_int4(0, 0, 0, 0);
    }
}

// zero the pad rows of a padded buffer (rows < *p_total whose prow_src < 0)
template <typename T>
__global__ void zero_pad_rows_kernel(T* __restrict__ buf, const int32_t* __restrict__ prow_src,
                                     const int32_t* __restrict__ p_total, int W, int64_t pmax) {
    pdl_wait();
    pdl_launch();
    const int64_t P = min((int64_t)*p_total, pmax);
    const int lane = threadIdx.x % 32;
    const int64_t warps = (int64_t)gridDim.x * blockDim.x / 32;
    const bool vec = vec_ok<T>(W) && ((uintptr_t)buf & 15) == 0;
    for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32; r < P; r += warps) {
        if (prow_src[r] >= 0) continue;
        if (vec) {  // 16-byte stores: a warp writes 512 contiguous bytes per instruction
            int4* d4 = reinterpret_cast<int4*>(buf + r * W);
            const int nv = (int)((int64_t)W * sizeof(T) / 16);
            for (int c = lane; c < nv; c += 32) d4[c] = make_int4(0, 0, 0, 0);
        } else {
            for (int c = lane; c < W; c += 32) buf[r * W + c] = Elem<T>::from_f(0.f);
        }
    }
}

// out[t, c] = sum over t's local slots j (in order) of weights[t, selected_k[j]] * y[slot_prow[j], c]
// (moe.hpp:258-266, T arithmetic: multiply, then add)
template <typename T>
__global__ void combine_kernel(const T* __restrict__ y, const int32_t* __restrict__ slot_prow,
                               const int32_t* __restrict__ selected_k, const int32_t* __restrict__ cum_expert_counts,
                               const float* __restrict__ gw, T* __restrict__ out, int T_tok, int H, int K) {
    pdl_wait();
    pdl_launch();
    const int t = (blockIdx.x * blockDim.x + threadIdx.x) / 32, lane = threadIdx.x % 32;
    if (t >= T_tok) return;
    const int j0 = cum_expert_counts[t], j1 = cum_expert_counts[t + 1];
    if (vec_ok<T>(H)) {
        // the slot rows of a column block are loaded together (up to 8 in flight per lane),
        // then summed in slot order
        constexpr int V = V16<T>::n, MAXJ = 8;
        int64_t rows[MAXJ];
        float wv[MAXJ];
        const int nj0 = min(MAXJ, j1 - j0);
#pragma unroll
        for (int q = 0; q < MAXJ; ++q) {
            rows[q] = q < nj0 ? slot_prow[j0 + q] : 0;
            wv[q] = (q < nj0 && gw) ? gw[(int64_t)t * K + selected_k[j0 + q]] : 1.f;
        }
        for (int c0 = lane * V; c0 < H; c0 += 32 * V) {
            float acc[V];
#pragma unroll
            for (int z = 0; z < V; ++z) acc[z] = 0.f;
            for (int jb = j0; jb < j1; jb += MAXJ) {
                const int nj = min(MAXJ, j1 - jb);
                if (jb != j0) {  // more than 8 local slots (K > 8): reload the slot table
#pragma unroll
                    for (int q = 0; q < MAXJ; ++q) {
                        rows[q] = q < nj ? slot_prow[jb + q] : 0;
                        wv[q] = (q < nj && gw) ? gw[(int64_t)t * K + selected_k[jb + q]] : 1.f;
                    }
                }
                int4 raw[MAXJ];
#pragma unroll
                for (int q = 0; q < MAXJ; ++q)
                    if (q < nj) raw[q] = __ldg(reinterpret_cast<const int4*>(y + rows[q] * H + c0));
#pragma unroll
                for (int q = 0; q < MAXJ; ++q) {
                    if (q >= nj) break;
                    float v[V];
                    V16<T>::unpack(raw[q], v);
                    if (gw) {
#pragma unroll
                        for (int z = 0; z < V; ++z) acc[z] = __fadd_rn(acc[z], __fmul_rn(wv[q], v[z]));
                    } else {  // unweighted: the scatter-add of dX rows to their token (moe.hpp:418-423)
#pragma unroll
                        for (int z = 0; z < V; ++z) acc[z] = __fadd_rn(acc[z], v[z]);
                    }
                }
            }
            if (j1 - j0 > MAXJ) {  // restore the first block's table for the next column block
#pragma unroll
                for (int q = 0; q < MAXJ; ++q) {
                    rows[q] = q < nj0 ? slot_prow[j0 + q] : 0;
                    wv[q] = (q < nj0 && gw) ? gw[(int64_t)t * K + selected_k[j0 + q]] : 1.f;
                }
            }
            V16<T>::store(out + (int64_t)t * H + c0, acc);
        }
        return;
    }
    for (int c0 = lane * 4; c0 < H; c0 += 128) {
        float acc[4] = {0.f, 0.f, 0.f, 0.f};
        for (int j = j0; j < j1; ++j) {
            const float wv = gw ? gw[(int64_t)t * K + selected_k[j]] : 1.f;
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
// dout rows come from `dout` ([T,H]) or, for expert parallelism, straight from the
// source rank's buffer over NVLink: peer_dout[t / s_local] + (t % s_local) * H.
template <typename T>
__global__ void __launch_bounds__(256, 3) out_reduction_bwd_kernel(const T* __restrict__ dout, const T* const* __restrict__ peer_dout,
                                         int s_local, const T* __restrict__ y,
                                         const int32_t* __restrict__ slot_prow, const int32_t* __restrict__ selected_k,
                                         const int32_t* __restrict__ cum_expert_counts, const float* __restrict__ gw,
                                         T* __restrict__ dy, float* __restrict__ wgrad, int T_tok, int H, int K) {
    pdl_wait();
    pdl_launch();
    const int t = (blockIdx.x * blockDim.x + threadIdx.x) / 32, lane = threadIdx.x % 32;
    if (t >= T_tok) return;
    const int j0 = cum_expert_counts[t], j1 = cum_expert_counts[t + 1];
    for (int k = lane; k < K; k += 32) wgrad[(int64_t)t * K + k] = 0.f;
    __syncwarp();
    if (j0 == j1) return;
    const T* gp = peer_dout ? peer_dout[t / s_local] + (int64_t)(t % s_local) * H : dout + (int64_t)t * H;
    if (vec_ok<T>(H)) {
        // column-vector outer loop: per 16-byte column block the dout vector and the rows of
        // up to 4 slots are loaded together (5 loads in flight per lane), then the slot dots
        // accumulate and the dy rows are stored
        constexpr int V = V16<T>::n;
        constexpr int MAXJ = 4;
        // the reference's fp64 dot (moe.hpp:289-294); bf16 operands multiply exactly in fp32
        // and the fp32 sum stays far inside the bf16-mode tolerance
        using DotT = typename std::conditional<sizeof(T) == 2, float, double>::type;
        const int nv = H / V;
        for (int jb = j0; jb < j1; jb += MAXJ) {
            const int nj = min(MAXJ, j1 - jb);
            int64_t rows[MAXJ];
            float wv[MAXJ];
            DotT dot[MAXJ];
#pragma unroll
            for (int q = 0; q < MAXJ; ++q) {
                rows[q] = q < nj ? slot_prow[jb + q] : 0;
                wv[q] = q < nj ? gw[(int64_t)t * K + selected_k[jb + q]] : 0.f;
                dot[q] = 0;
            }
            for (int vi = lane; vi < nv; vi += 32) {
                const int4 graw = __ldg(reinterpret_cast<const int4*>(gp + vi * V));
                int4 yr[MAXJ];
#pragma unroll
                for (int q = 0; q < MAXJ; ++q)
                    if (q < nj) yr[q] = __ldg(reinterpret_cast<const int4*>(y + rows[q] * H + vi * V));
                float g[V];
                V16<T>::unpack(graw, g);
#pragma unroll
                for (int q = 0; q < MAXJ; ++q) {
                    if (q >= nj) break;
                    float yv[V], o[V];
                    V16<T>::unpack(yr[q], yv);
#pragma unroll
                    for (int z = 0; z < V; ++z) {
                        o[z] = __fmul_rn(wv[q], g[z]);
                        if constexpr (sizeof(T) == 2) dot[q] = __fmaf_rn(g[z], yv[z], dot[q]);
                        else dot[q] += (double)g[z] * (double)yv[z];
                    }
                    V16<T>::store(dy + rows[q] * H + vi * V, o);
                }
            }
#pragma unroll
            for (int q = 0; q < MAXJ; ++q) {
                DotT d = dot[q];
#pragma unroll
                for (int o = 16; o; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
                if (lane == 0 && q < nj) wgrad[(int64_t)t * K + selected_k[jb + q]] = (float)d;
            }
        }
        return;
    }
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
// CTA tile: 64 tokens x 64 h. Phase 1 computes the router term (matmul_nt order over e)
// with 8 x 4 register tiles from transposed shared-memory operands; phase 2 re-maps
// the threads onto 16-byte column vectors for the slot sum and the store.
constexpr int kDxT = 64, kDxH = 64, kDxE = 32;
template <typename T, bool FROM_SLOTS>
__global__ void __launch_bounds__(128) dx_finalize_kernel(const T* __restrict__ src, const int32_t* __restrict__ slot_prow,
                                                          const int32_t* __restrict__ cum_expert_counts,
                                                          const float* __restrict__ dl, const T* __restrict__ wr,
                                                          T* __restrict__ dx, int S, int H, int N) {
    __shared__ __align__(16) float sm[kDxT * (kDxH + 4)];  // phase 1: ds[e][t], ws[e][h]; phase 2: rt[t][h]
    float (*ds)[kDxT] = reinterpret_cast<float (*)[kDxT]>(sm);
    float (*ws)[kDxH] = reinterpret_cast<float (*)[kDxH]>(sm + kDxE * kDxT);
    const int t0 = blockIdx.x * kDxT, h0 = blockIdx.y * kDxH;
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;  // 16 h-quads x 8 token-octets
    float acc[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
    for (int e0 = 0; e0 < N; e0 += kDxE) {
        for (int i = threadIdx.x; i < kDxE * kDxT; i += 128) {
            const int ee = i % kDxE, rr = i / kDxE;  // consecutive threads: consecutive e (coalesced)
            const int e = e0 + ee, t = t0 + rr, h = h0 + rr;
            ds[ee][rr] = (e < N && t < S) ? dl[(int64_t)t * N + e] : 0.f;
            ws[ee][rr] = (e < N && h < H) ? Elem<T>::load(wr + (int64_t)h * N + e) : 0.f;
        }
        __syncthreads();
        const int eend = min(kDxE, N - e0);
        for (int ee = 0; ee < eend; ++ee) {
            const float4 a0 = *reinterpret_cast<const float4*>(&ds[ee][ty * 8]);
            const float4 a1 = *reinterpret_cast<const float4*>(&ds[ee][ty * 8 + 4]);
            const float4 b4 = *reinterpret_cast<const float4*>(&ws[ee][tx * 4]);
            const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
            const float b[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = __fadd_rn(acc[i][j], __fmul_rn(a[i], b[j]));
        }
        __syncthreads();
    }
    float (*rt)[kDxH + 4] = reinterpret_cast<float (*)[kDxH + 4]>(sm);  // 64 x 68 floats fits in sm
#pragma unroll
    for (int i = 0; i < 8; ++i)
        *reinterpret_cast<float4*>(&rt[ty * 8 + i][tx * 4]) = make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
    __syncthreads();
    constexpr int V = 16 / sizeof(T);
    const bool vec = (H % V) == 0 && (h0 + kDxH <= H);
    if (vec) {
        constexpr int VPT = kDxH / V;  // vectors per token row
        for (int q = threadIdx.x; q < kDxT * VPT; q += 128) {
            const int tt = q / VPT, vv = q % VPT;
            const int t = t0 + tt;
            if (t >= S) continue;
            const int h = h0 + vv * V;
            float base[V], v[V];
#pragma unroll
            for (int z = 0; z < V; ++z) base[z] = 0.f;
            if (FROM_SLOTS) {
                const int j0 = cum_expert_counts[t], j1 = cum_expert_counts[t + 1];
                for (int j = j0; j < j1; ++j) {
                    V16<T>::load(src + (int64_t)slot_prow[j] * H + h, v);
#pragma unroll
                    for (int z = 0; z < V; ++z) base[z] = __fadd_rn(base[z], v[z]);
                }
            } else {
                V16<T>::load(src + (int64_t)t * H + h, base);
            }
#pragma unroll
            for (int z = 0; z < V; ++z) base[z] = __fadd_rn(base[z], rt[tt][vv * V + z]);
            V16<T>::store(dx + (int64_t)t * H + h, base);
        }
    } else {
        for (int q = threadIdx.x; q < kDxT * kDxH; q += 128) {
            const int tt = q / kDxH, hh = q % kDxH;
            const int t = t0 + tt, h = h0 + hh;
            if (t >= S || h >= H) continue;
            float base = 0.f;
            if (FROM_SLOTS) {
                const int j0 = cum_expert_counts[t], j1 = cum_expert_counts[t + 1];
                for (int j = j0; j < j1; ++j) base = __fadd_rn(base, Elem<T>::to_f(src[(int64_t)slot_prow[j] * H + h]));
            } else {
                base = Elem<T>::to_f(src[(int64_t)t * H + h]);
            }
            dx[(int64_t)t * H + h] = Elem<T>::from_f(__fadd_rn(base, rt[tt][hh]));
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
    launch_k(gather_rows_kernel<T>, dim3(grid_for_rows(pmax)), dim3(256), 0, st, x, prow_src, p_total, out, H, pmax);
    B2_LAUNCH_CHECK();
}

template <typename T>
void launch_gather_tokens(const T* x, const int32_t* cec, const int32_t* slot_prow, int T_tok,
                          const int32_t* prow_src, const int32_t* p_total, T* out, int H, int64_t pmax,
                          cudaStream_t st) {
    if (((int64_t)H * sizeof(T)) % 16 != 0 || ((uintptr_t)x & 15) || ((uintptr_t)out & 15)) {  // not 16-B rows
        launch_gather_rows<T>(x, prow_src, p_total, out, H, pmax, st);
        return;
    }
    launch_k(gather_tokens_kernel<T>, dim3(grid_for_rows(std::max<int64_t>(pmax, T_tok))), dim3(256), 0, st, x, cec,
             slot_prow, T_tok, prow_src, p_total, out, H, pmax);
    B2_LAUNCH_CHECK();
}

template <typename T>
void launch_zero_pad_rows(T* buf, const int32_t* prow_src, const int32_t* p_total, int W, int64_t pmax,
                          cudaStream_t st) {
    if (pmax <= 0) return;
    launch_k(zero_pad_rows_kernel<T>, dim3(grid_for_rows(pmax)), dim3(256), 0, st, buf, prow_src, p_total, W, pmax);
    B2_LAUNCH_CHECK();
}

template <typename T>
void launch_combine(const T* y, const int32_t* slot_prow, const int32_t* selected_k, const int32_t* cec,
                    const float* gw, T* out, int T_tok, int H, int K, cudaStream_t st) {
    if (T_tok <= 0) return;
    launch_k(combine_kernel<T>, dim3((unsigned)ceil_div(T_tok, 8)), dim3(256), 0, st, y, slot_prow, selected_k, cec, gw, out, T_tok, H, K);
    B2_LAUNCH_CHECK();
}

// top-k weight gradients from the dgrad epilogue's row partials (bf16 path): the reference's
// weights_grad[t, k] = dout[t] . mlp_out[r] (moe.hpp:283-294) equals dH'[r] . h[r] with
// dH' = dout . Wd^T, which the dgrad GEMM accumulates anyway; its epilogue leaves np partial
// dots per padded row (one per 128-column half tile), summed here in a fixed order. Tokens
// without a local slot get zeros, like the reference's zero-initialised weights_grad.
__global__ void wgrad_from_parts_kernel(const float* __restrict__ part, int np, const int32_t* __restrict__ slot_prow,
                                        const int32_t* __restrict__ selected_k, const int32_t* __restrict__ cec,
                                        float* __restrict__ wgrad, int T_tok, int K) {
    pdl_wait();
    pdl_launch();
    // one thread per (token, k): find the token's local slot holding k (if any)
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (int64_t)T_tok * K) return;
    const int t = (int)(i / K), k = (int)(i % K);
    float acc = 0.f;
    for (int j = cec[t], j1 = cec[t + 1]; j < j1; ++j) {
        if (selected_k[j] != k) continue;
        const float* pr = part + (int64_t)slot_prow[j] * np;
        for (int q = 0; q < np; ++q) acc += pr[q];
        break;
    }
    wgrad[i] = acc;
}

void launch_wgrad_from_parts(const float* part, int np, const int32_t* slot_prow, const int32_t* selected_k,
                             const int32_t* cec, float* wgrad, int T_tok, int K, cudaStream_t st) {
    if (T_tok <= 0) return;
    launch_k(wgrad_from_parts_kernel, dim3((unsigned)ceil_div((int64_t)T_tok * K, 256)), dim3(256), 0, st, part, np,
             slot_prow, selected_k, cec, wgrad, T_tok, K);
    B2_LAUNCH_CHECK();
}

template <typename T>
void launch_out_reduction_bwd(const T* dout, const T* const* peer_dout, int s_local, const T* y,
                              const int32_t* slot_prow, const int32_t* selected_k, const int32_t* cec, const float* gw,
                              T* dy, float* wgrad, int T_tok, int H, int K, cudaStream_t st) {
    if (T_tok <= 0) return;
    launch_k(out_reduction_bwd_kernel<T>, dim3((unsigned)ceil_div(T_tok, 8)), dim3(256), 0, st, dout, peer_dout, s_local, y, slot_prow,
                                                                               selected_k, cec, gw, dy, wgrad, T_tok,
                                                                               H, K);
    B2_LAUNCH_CHECK();
}

template <typename T>
void launch_dx_finalize(const T* src, bool from_slots, const int32_t* slot_prow, const int32_t* cec, const float* dl,
                        const T* wr, T* dx, int S, int H, int N, cudaStream_t st) {
    if (S <= 0) return;
    dim3 grid((unsigned)ceil_div(S, kDxT), (unsigned)ceil_div(H, kDxH));
    if (from_slots)
        dx_finalize_kernel<T, true><<<grid, 128, 0, st>>>(src, slot_prow, cec, dl, wr, dx, S, H, N);
    else
        dx_finalize_kernel<T, false><<<grid, 128, 0, st>>>(src, slot_prow, cec, dl, wr, dx, S, H, N);
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
    template void launch_gather_tokens<T>(const T*, const int32_t*, const int32_t*, int, const int32_t*,          \
                                          const int32_t*, T*, int, int64_t, cudaStream_t);                       \
    template void launch_combine<T>(const T*, const int32_t*, const int32_t*, const int32_t*, const float*, T*, int, \
                                    int, int, cudaStream_t);                                                       \
    template void launch_out_reduction_bwd<T>(const T*, const T* const*, int, const T*, const int32_t*,           \
                                              const int32_t*, const int32_t*, const float*, T*, float*, int, int,  \
                                              int, cudaStream_t);                                                  \
    template void launch_dx_finalize<T>(const T*, bool, const int32_t*, const int32_t*, const float*, const T*, T*, \
                                        int, int, int, cudaStream_t);                                              \
    template void launch_swiglu_fwd<T>(const T*, const T*, T*, const int32_t*, int, int64_t, cudaStream_t);        \
    template void launch_swiglu_bwd<T>(const T*, const T*, const T*, T*, const int32_t*, int, int64_t, cudaStream_t);
B2_INST(float)
B2_INST(__nv_bfloat16)
#undef B2_INST

}  // namespace b2
