// Expert-parallel token dispatch / combine around the expert MLP (EP > 1).
//
// The reference gathers every rank's tokens on every rank (allgather, moe.hpp:365-367)
// and returns the combined rows with a rank-ordered reducescatter (moe.hpp:378); the
// backward mirrors both (moe.hpp:400, 427-428). Here a token is sent only to the ranks
// that host at least one of its top-k experts (dedup per destination), as an
// all-to-all-v over NVLink (comm.cpp all_to_all_v):
//   plan     one CTA scans, per destination rank r in order, the tokens that route to r
//            (token order) -> send position, counts and offsets (destination-major).
//   pack     token rows (16-byte vectors) + a metadata row {t, top-k ids, top-k weights}.
//   receive  rows arrive ordered by (source rank, source token): exactly the reference's
//            gathered order src*S + t restricted to the tokens this rank needs, so the
//            stable expert-sorted permutation is unchanged (SURVEY §8 e).
//   return   the source sums the partial rows sent back by each destination in rank
//            order (the reducescatter's member order, comm.hpp:391-394); ranks with no
//            expert for a token contribute an exact zero in the reference.
#include "b2_common.cuh"
#include "kernels.h"

namespace b2 {

__device__ __forceinline__ int warp_incl_scan_i(int x, int lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    return x;
}

// one CTA: send_pos[r*S + t] (position within destination r, or -1), send_cnt[r], send_off[r]
__global__ void __launch_bounds__(1024) dest_plan_kernel(const int32_t* __restrict__ gi, int S, int K, int E, int NR,
                                                         int32_t* __restrict__ send_pos, int32_t* __restrict__ send_cnt,
                                                         int32_t* __restrict__ send_off) {
    __shared__ int wsum[32];
    const int lane = threadIdx.x % 32, warp = threadIdx.x / 32, nw = blockDim.x / 32;
    int off = 0;
    for (int r = 0; r < E; ++r) {
        int carry = 0;
        for (int base = 0; base < S; base += blockDim.x) {
            const int t = base + threadIdx.x;
            int f = 0;
            if (t < S)
                for (int k = 0; k < K; ++k) f |= (gi[(int64_t)t * K + k] / NR) == r;
            const int x = warp_incl_scan_i(f, lane);
            if (lane == 31) wsum[warp] = x;
            __syncthreads();
            if (warp == 0) {
                const int s = lane < nw ? wsum[lane] : 0;
                const int si = warp_incl_scan_i(s, lane);
                if (lane < nw) wsum[lane] = si;
            }
            __syncthreads();
            const int excl = carry + (warp > 0 ? wsum[warp - 1] : 0) + x - f;
            if (t < S) send_pos[(int64_t)r * S + t] = f ? excl : -1;
            carry += wsum[nw - 1];
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            send_cnt[r] = carry;
            send_off[r] = off;
        }
        off += carry;
    }
}

// warp per token: copy the row to every destination slot (+ metadata when meta != null)
template <typename T>
__global__ void pack_rows_kernel(const T* __restrict__ x, const int32_t* __restrict__ send_pos,
                                 const int32_t* __restrict__ send_off, int S, int E, int H, T* __restrict__ send_x,
                                 const int32_t* __restrict__ gi, const float* __restrict__ gw, int K,
                                 int32_t* __restrict__ meta) {
    const int t = (blockIdx.x * blockDim.x + threadIdx.x) / 32, lane = threadIdx.x % 32;
    if (t >= S) return;
    const int MW = 1 + 2 * K;
    for (int r = 0; r < E; ++r) {
        const int pos = send_pos[(int64_t)r * S + t];
        if (pos < 0) continue;
        const int64_t row = (int64_t)send_off[r] + pos;
        if (((int64_t)H * sizeof(T)) % 16 == 0) {
            const int nv = (int)((int64_t)H * sizeof(T) / 16);
            const int4* s4 = reinterpret_cast<const int4*>(x + (int64_t)t * H);
            int4* d4 = reinterpret_cast<int4*>(send_x + row * H);
            for (int v = lane; v < nv; v += 32) d4[v] = __ldg(s4 + v);
        } else {
            for (int c = lane; c < H; c += 32) send_x[row * H + c] = x[(int64_t)t * H + c];
        }
        if (meta) {
            int32_t* m = meta + row * MW;
            if (lane == 0) m[0] = t;
            for (int k = lane; k < K; k += 32) {
                m[1 + k] = gi[(int64_t)t * K + k];
                m[1 + K + k] = __float_as_int(gw[(int64_t)t * K + k]);
            }
        }
    }
}

__global__ void unpack_meta_kernel(const int32_t* __restrict__ meta, int64_t n, int K, int32_t* __restrict__ gi,
                                   float* __restrict__ gw, int32_t* __restrict__ src_t) {
    const int MW = 1 + 2 * K;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t* m = meta + i * MW;
        src_t[i] = m[0];
        for (int k = 0; k < K; ++k) {
            gi[i * K + k] = m[1 + k];
            gw[i * K + k] = __int_as_float(m[1 + K + k]);
        }
    }
}

// out[t] = sum over destinations r (in rank order) that received t of ret[send_off[r] + pos]
template <typename T>
__global__ void return_sum_kernel(const T* __restrict__ ret, const int32_t* __restrict__ send_pos,
                                  const int32_t* __restrict__ send_off, int S, int E, int W, T* __restrict__ out) {
    const int t = (blockIdx.x * blockDim.x + threadIdx.x) / 32, lane = threadIdx.x % 32;
    if (t >= S) return;
    for (int c = lane; c < W; c += 32) {
        float acc = 0.f;
        bool any = false;
        for (int r = 0; r < E; ++r) {
            const int pos = send_pos[(int64_t)r * S + t];
            if (pos < 0) continue;
            const float v = Elem<T>::to_f(ret[((int64_t)send_off[r] + pos) * W + c]);
            acc = any ? __fadd_rn(acc, v) : v;
            any = true;
        }
        out[(int64_t)t * W + c] = Elem<T>::from_f(acc);
    }
}

// vectorised variant for 16-byte aligned rows
template <typename T>
__global__ void return_sum_vec_kernel(const T* __restrict__ ret, const int32_t* __restrict__ send_pos,
                                      const int32_t* __restrict__ send_off, int S, int E, int W, T* __restrict__ out) {
    const int t = (blockIdx.x * blockDim.x + threadIdx.x) / 32, lane = threadIdx.x % 32;
    if (t >= S) return;
    constexpr int V = 16 / sizeof(T);
    const int nv = W / V;
    for (int v = lane; v < nv; v += 32) {
        float acc[V];
#pragma unroll
        for (int q = 0; q < V; ++q) acc[q] = 0.f;
        bool any = false;
        for (int r = 0; r < E; ++r) {
            const int pos = send_pos[(int64_t)r * S + t];
            if (pos < 0) continue;
            const int4 raw = __ldg(reinterpret_cast<const int4*>(ret + ((int64_t)send_off[r] + pos) * W) + v);
            float f[V];
            if constexpr (sizeof(T) == 4) {
                f[0] = __int_as_float(raw.x);
                f[1] = __int_as_float(raw.y);
                f[2] = __int_as_float(raw.z);
                f[3] = __int_as_float(raw.w);
            } else {
                const uint32_t w[4] = {(uint32_t)raw.x, (uint32_t)raw.y, (uint32_t)raw.z, (uint32_t)raw.w};
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    f[2 * q] = __uint_as_float(w[q] << 16);
                    f[2 * q + 1] = __uint_as_float(w[q] & 0xFFFF0000u);
                }
            }
#pragma unroll
            for (int q = 0; q < V; ++q) acc[q] = any ? __fadd_rn(acc[q], f[q]) : f[q];
            any = true;
        }
        int4 o;
        if constexpr (sizeof(T) == 4) {
            o = make_int4(__float_as_int(acc[0]), __float_as_int(acc[1]), __float_as_int(acc[2]), __float_as_int(acc[3]));
        } else {
            uint32_t w[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                __nv_bfloat162 b = __floats2bfloat162_rn(acc[2 * q], acc[2 * q + 1]);
                w[q] = *reinterpret_cast<uint32_t*>(&b);
            }
            o = make_int4((int)w[0], (int)w[1], (int)w[2], (int)w[3]);
        }
        reinterpret_cast<int4*>(out + (int64_t)t * W)[v] = o;
    }
}

void launch_dest_plan(const int32_t* gi, int S, int K, int E, int NR, int32_t* send_pos, int32_t* send_cnt,
                      int32_t* send_off, cudaStream_t st) {
    dest_plan_kernel<<<1, 1024, 0, st>>>(gi, S, K, E, NR, send_pos, send_cnt, send_off);
    B2_LAUNCH_CHECK();
}

template <typename T>
void launch_pack_rows(const T* x, const int32_t* send_pos, const int32_t* send_off, int S, int E, int H, T* send_x,
                      const int32_t* gi, const float* gw, int K, int32_t* meta, cudaStream_t st) {
    if (S <= 0) return;
    pack_rows_kernel<T><<<(unsigned)ceil_div(S, 8), 256, 0, st>>>(x, send_pos, send_off, S, E, H, send_x, gi, gw, K,
                                                                   meta);
    B2_LAUNCH_CHECK();
}

void launch_unpack_meta(const int32_t* meta, int64_t n, int K, int32_t* gi, float* gw, int32_t* src_t,
                        cudaStream_t st) {
    if (n <= 0) return;
    unpack_meta_kernel<<<(unsigned)std::min<int64_t>(1184, ceil_div(n, 256)), 256, 0, st>>>(meta, n, K, gi, gw, src_t);
    B2_LAUNCH_CHECK();
}

template <typename T>
void launch_return_sum(const T* ret, const int32_t* send_pos, const int32_t* send_off, int S, int E, int W, T* out,
                       cudaStream_t st) {
    if (S <= 0) return;
    if (((int64_t)W * sizeof(T)) % 16 == 0)
        return_sum_vec_kernel<T><<<(unsigned)ceil_div(S, 8), 256, 0, st>>>(ret, send_pos, send_off, S, E, W, out);
    else
        return_sum_kernel<T><<<(unsigned)ceil_div(S, 8), 256, 0, st>>>(ret, send_pos, send_off, S, E, W, out);
    B2_LAUNCH_CHECK();
}

#define B2_EP_INST(T)                                                                                              \
    template void launch_pack_rows<T>(const T*, const int32_t*, const int32_t*, int, int, int, T*, const int32_t*, \
                                      const float*, int, int32_t*, cudaStream_t);                                  \
    template void launch_return_sum<T>(const T*, const int32_t*, const int32_t*, int, int, int, T*, cudaStream_t);
B2_EP_INST(float)
B2_EP_INST(__nv_bfloat16)
#undef B2_EP_INST

}  // namespace b2
