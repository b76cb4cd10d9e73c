// Token counting and index generation (Algorithm 1 stages 2-3) on the gathered
// routing table, bit-exact with the reference.
//
// Reference: count_tokens (include/optimus/moe.hpp:122-164) and generate_indices
// (moe.hpp:167-197). The reference's result is a STABLE sort of the local
// selections by expert, in (token, k) order within an expert, independent of the
// token-block size (test_moe.cpp:130-207). Here:
//   1. one warp per 64-token chunk builds a shared-memory histogram of its local
//      selections (counts are order-free, so smem atomics are deterministic) and the
//      per-token local counts;
//   2. one CTA scans: each warp walks one expert's chunk histogram (contiguous,
//      expert-major) giving every (expert, chunk) its first row inside the expert;
//      a warp scan over the expert totals gives cum_token_counts and the 128-row
//      padded group starts the GEMMs use; a tiled block scan gives cum_expert_counts;
//   3. each warp re-walks its chunk in (t, k) order in 32-entry batches and ranks
//      equal experts with __match_any_sync plus a per-expert carry, so the row of
//      every selection equals the reference's counter(ln, tid)++.
// The TBS-blocked diagnostics (partial_token_counts / partial_cum / counter,
// moe.hpp:148-158) do not feed any later stage; they are produced only when the
// artifacts are exported (launch_partial_counts).
#include "b2_common.cuh"
#include "kernels.h"

namespace b2 {

constexpr int kChunk = 64;  // tokens per warp chunk
constexpr int kWarpsPerCta = 4;

__device__ __forceinline__ int local_of(int e, int n_start, int nr) {
    return (e >= n_start && e < n_start + nr) ? e - n_start : -1;
}

// 1. histograms (whist [nr][nchunks]) + per-token local counts
__global__ void count_kernel(const int32_t* __restrict__ gidx, int T, int K, int N, int n_start, int nr,
                             int nchunks, int32_t* __restrict__ whist, int32_t* __restrict__ expert_counts,
                             int32_t* __restrict__ err) {
    pdl_wait();
    pdl_launch();
    extern __shared__ int32_t sh[];  // [kWarpsPerCta][nr]
    const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int chunk = blockIdx.x * kWarpsPerCta + w;
    int32_t* hist = sh + w * nr;
    for (int i = lane; i < nr; i += 32) hist[i] = 0;
    __syncwarp();
    const int t0 = chunk * kChunk;
    if (t0 < T) {
        const int t1 = min(T, t0 + kChunk);
        const int nent = (t1 - t0) * K;
        for (int f = lane; f < nent; f += 32) {
            const int e = gidx[(int64_t)t0 * K + f];
            if (e < 0 || e >= N) {
                atomicExch(err, 1);
                continue;
            }
            const int ln = local_of(e, n_start, nr);
            if (ln >= 0) atomicAdd(&hist[ln], 1);
        }
        for (int t = t0 + lane; t < t1; t += 32) {
            int c = 0;
            for (int k = 0; k < K; ++k) c += local_of(gidx[(int64_t)t * K + k], n_start, nr) >= 0;
            expert_counts[t] = c;
        }
    }
    __syncwarp();
    if (chunk < nchunks)
        for (int i = lane; i < nr; i += 32) whist[(int64_t)i * nchunks + chunk] = hist[i];
}

__device__ __forceinline__ int warp_incl_scan(int x, int lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    return x;
}

// exclusive block scan (R consecutive elements per thread and round); returns the total
template <class Get, class Put>
__device__ int64_t block_scan(int64_t n, Get get, Put put, int* wsum) {
    // each thread owns R consecutive elements per round: a serial local scan, one block
    // scan of the thread totals, then the R exclusive prefixes (integer: order-independent)
    constexpr int R = 16;
    const int lane = threadIdx.x % 32, warp = threadIdx.x / 32, nw = blockDim.x / 32;
    int64_t carry = 0;
    for (int64_t base = 0; base < n; base += (int64_t)blockDim.x * R) {
        const int64_t i0 = base + (int64_t)threadIdx.x * R;
        int v[R];
        int tsum = 0;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            v[r] = i0 + r < n ? get(i0 + r) : 0;
            tsum += v[r];
        }
        const int x = warp_incl_scan(tsum, lane);
        if (lane == 31) wsum[warp] = x;
        __syncthreads();
        if (warp == 0) {
            const int s = lane < nw ? wsum[lane] : 0;
            const int si = warp_incl_scan(s, lane);
            if (lane < nw) wsum[lane] = si;
        }
        __syncthreads();
        int64_t excl = carry + (warp > 0 ? wsum[warp - 1] : 0) + x - tsum;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            if (i0 + r < n) put(i0 + r, excl);
            excl += v[r];
        }
        carry += wsum[nw - 1];
        __syncthreads();
    }
    return carry;
}

// block_scan over an int32 array with 16-byte loads and stores (in, out 16-byte aligned; the
// last partial group of 16 element-wise)
__device__ int64_t block_scan_i32(const int32_t* __restrict__ in, int32_t* __restrict__ out, int64_t n, int* wsum) {
    constexpr int R = 16;
    const int lane = threadIdx.x % 32, warp = threadIdx.x / 32, nw = blockDim.x / 32;
    int64_t carry = 0;
    for (int64_t base = 0; base < n; base += (int64_t)blockDim.x * R) {
        const int64_t i0 = base + (int64_t)threadIdx.x * R;
        int v[R];
        if (i0 + R <= n) {
#pragma unroll
            for (int q = 0; q < R / 4; ++q) {
                const int4 w = *reinterpret_cast<const int4*>(in + i0 + 4 * q);
                v[4 * q] = w.x;
                v[4 * q + 1] = w.y;
                v[4 * q + 2] = w.z;
                v[4 * q + 3] = w.w;
            }
        } else {
#pragma unroll
            for (int r = 0; r < R; ++r) v[r] = i0 + r < n ? in[i0 + r] : 0;
        }
        int tsum = 0;
#pragma unroll
        for (int r = 0; r < R; ++r) tsum += v[r];
        const int x = warp_incl_scan(tsum, lane);
        if (lane == 31) wsum[warp] = x;
        __syncthreads();
        if (warp == 0) {
            const int s = lane < nw ? wsum[lane] : 0;
            const int si = warp_incl_scan(s, lane);
            if (lane < nw) wsum[lane] = si;
        }
        __syncthreads();
        int excl = (int)carry + (warp > 0 ? wsum[warp - 1] : 0) + x - tsum;
        int o[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            o[r] = excl;
            excl += v[r];
        }
        if (i0 + R <= n) {
#pragma unroll
            for (int q = 0; q < R / 4; ++q)
                *reinterpret_cast<int4*>(out + i0 + 4 * q) = make_int4(o[4 * q], o[4 * q + 1], o[4 * q + 2], o[4 * q + 3]);
        } else {
#pragma unroll
            for (int r = 0; r < R; ++r)
                if (i0 + r < n) out[i0 + r] = o[r];
        }
        carry += wsum[nw - 1];
        __syncthreads();
    }
    return carry;
}

// 2. scans, one CTA of 1024 threads
__global__ void __launch_bounds__(1024) scan_kernel(const int32_t* __restrict__ whist, int nchunks, int nr,
                                                    const int32_t* __restrict__ expert_counts, int T,
                                                    int32_t* __restrict__ wbase /*[nr][nchunks]*/,
                                                    int32_t* __restrict__ token_counts,
                                                    int32_t* __restrict__ cum_token_counts,
                                                    int32_t* __restrict__ pad_start,
                                                    int32_t* __restrict__ cum_expert_counts,
                                                    int32_t* __restrict__ expert_order) {
    pdl_wait();
    pdl_launch();
    extern __shared__ int32_t tot[];  // [nr]
    __shared__ int wsum[32];
    const int lane = threadIdx.x % 32, warp = threadIdx.x / 32, nw = blockDim.x / 32;
    // (a) within-expert chunk offsets (expert-major, chunk-minor == the reference's
    //     partial_cum order restricted to whole chunks). With fewer experts than warps (EP:
    //     nr = N / EP over a table EP times longer) each expert's chunks are split into
    //     segments over wpe warps, then every segment adds the totals of the ones before it
    __shared__ int segsum[32];
    const int wpe = nr >= nw ? 1 : nw / nr;           // warps per expert
    const int ngroups = nw / wpe;                     // experts in flight
    const int seg = (int)ceil_div(nchunks, wpe);      // chunks per warp segment
    for (int e0 = 0; e0 < nr; e0 += ngroups) {
        const int ln = e0 + warp / wpe, sg = warp % wpe;
        const bool active = warp < ngroups * wpe && ln < nr;
        const int c0 = sg * seg, c1 = min(nchunks, c0 + seg);
        int carry = 0;
        if (active) {
            const int32_t* hrow = whist + (int64_t)ln * nchunks;
            int32_t* brow = wbase + (int64_t)ln * nchunks;
            constexpr int P = 8;  // 8 x 32 chunk counts loaded together, then scanned in order
            for (int cb = c0; cb < c1; cb += 32 * P) {
                int vv[P];
#pragma unroll
                for (int q = 0; q < P; ++q) {
                    const int c = cb + 32 * q + lane;
                    vv[q] = c < c1 ? hrow[c] : 0;
                }
#pragma unroll
                for (int q = 0; q < P; ++q) {
                    const int c = cb + 32 * q + lane;
                    const int x = warp_incl_scan(vv[q], lane);
                    if (c < c1) brow[c] = carry + x - vv[q];
                    carry += __shfl_sync(0xffffffffu, x, 31);
                }
            }
        }
        if (wpe > 1) {
            if (lane == 0) segsum[warp] = active ? carry : 0;
            __syncthreads();
            if (active) {
                int off = 0;
                for (int q = 0; q < sg; ++q) off += segsum[warp - sg + q];
                if (off) {
                    int32_t* brow = wbase + (int64_t)ln * nchunks;
                    for (int c = c0 + lane; c < c1; c += 32) brow[c] += off;
                }
                if (sg == wpe - 1 && lane == 0) tot[ln] = off + carry;
            }
            __syncthreads();
        } else if (active && lane == 0) {
            tot[ln] = carry;
        }
    }
    __syncthreads();
    // (b) expert boundaries and padded starts (warp 0)
    if (warp == 0) {
        int carry = 0, pcarry = 0;
        for (int l0 = 0; l0 < nr; l0 += 32) {
            const int ln = l0 + lane;
            const int v = ln < nr ? tot[ln] : 0;
            const int pv = (int)round_up(v, kRowAlign);
            const int x = warp_incl_scan(v, lane), px = warp_incl_scan(pv, lane);
            if (ln < nr) {
                token_counts[ln] = v;
                cum_token_counts[ln] = carry + x - v;
                pad_start[ln] = pcarry + px - pv;
            }
            carry += __shfl_sync(0xffffffffu, x, 31);
            pcarry += __shfl_sync(0xffffffffu, px, 31);
        }
        if (lane == 0) {
            cum_token_counts[nr] = carry;
            pad_start[nr] = pcarry;
        }
    }
    // (b') the experts by descending row count, ties by index: the weight-gradient GEMMs take
    //      their per-expert tiles (K extent = the expert's rows) in this order, so the persistent
    //      CTAs' static tile stride spreads the longest tiles first (an LPT-like schedule)
    if (expert_order)
        for (int e = threadIdx.x; e < nr; e += blockDim.x) {
            const int ce = tot[e];
            int r = 0;
            for (int j = 0; j < nr; ++j) r += (tot[j] > ce) || (tot[j] == ce && j < e);
            expert_order[r] = e;
        }
    // (c) cum_expert_counts: exclusive scan of the per-token local counts (16 per thread per
    //     round, moved as 16-byte vectors: the table is EP times longer than the local tokens)
    const int64_t te = block_scan_i32(expert_counts, cum_expert_counts, T, wsum);
    if (threadIdx.x == 0) cum_expert_counts[T] = (int32_t)te;
}

// 3. stable scatter
__global__ void scatter_kernel(const int32_t* __restrict__ gidx, int T, int K, int n_start, int nr, int nchunks,
                               const int32_t* __restrict__ wbase, const int32_t* __restrict__ cum_token_counts,
                               const int32_t* __restrict__ pad_start, const int32_t* __restrict__ cum_expert_counts,
                               int32_t* __restrict__ input_indices, int32_t* __restrict__ output_indices,
                               int32_t* __restrict__ selected_k, int32_t* __restrict__ slot_prow,
                               int32_t* __restrict__ prow_src, const float* __restrict__ gw,
                               float* __restrict__ prow_w) {
    pdl_wait();
    pdl_launch();
    extern __shared__ int32_t sh[];  // carry [kWarpsPerCta][nr] (row offset inside the expert)
    const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int chunk = blockIdx.x * kWarpsPerCta + w;
    const int t0 = chunk * kChunk;
    if (t0 >= T) return;
    int32_t* carry = sh + w * nr;
    for (int i = lane; i < nr; i += 32) carry[i] = wbase[(int64_t)i * nchunks + chunk];
    __syncwarp();
    const int t1 = min(T, t0 + kChunk);
    const int nent = (t1 - t0) * K;
    const unsigned lt = (1u << lane) - 1u;
    for (int f0 = 0; f0 < nent; f0 += 32) {
        const int f = f0 + lane;
        const bool valid = f < nent;
        const int t = t0 + (valid ? f / K : 0), k = valid ? f % K : 0;
        const int e = valid ? gidx[(int64_t)t * K + k] : -1;
        const int ln = valid ? local_of(e, n_start, nr) : -1;
        const unsigned peers = __match_any_sync(0xffffffffu, ln);
        int off = 0;
        if (ln >= 0) off = carry[ln] + __popc(peers & lt);
        __syncwarp();
        if (ln >= 0 && (peers & lt) == 0) carry[ln] += __popc(peers);  // group leader
        __syncwarp();
        if (ln >= 0) {
            int before = 0;  // local selections of token t with k' < k
            for (int kk = 0; kk < k; ++kk) before += local_of(gidx[(int64_t)t * K + kk], n_start, nr) >= 0;
            const int pos = cum_expert_counts[t] + before;
            const int row = cum_token_counts[ln] + off;
            const int prow = pad_start[ln] + off;
            input_indices[row] = t;
            output_indices[pos] = row;
            selected_k[pos] = k;
            slot_prow[pos] = prow;
            prow_src[prow] = t;
            if (prow_w) prow_w[prow] = gw[(int64_t)t * K + k];
        }
    }
}

// pad rows of each expert group read as zero tokens
__global__ void pad_fill_kernel(const int32_t* __restrict__ token_counts, const int32_t* __restrict__ pad_start,
                                int nr, int32_t* __restrict__ prow_src, float* __restrict__ prow_w) {
    pdl_wait();
    pdl_launch();
    const int ln = blockIdx.x;
    const int b = pad_start[ln] + token_counts[ln], e = pad_start[ln + 1];
    for (int r = b + threadIdx.x; r < e; r += blockDim.x) {
        prow_src[r] = -1;
        if (prow_w) prow_w[r] = 0.f;
    }
}

void launch_routing_index(const RoutingIndexArgs& a, cudaStream_t st) {
    const int nchunks = (int)ceil_div(a.T, kChunk);
    const int nblk = (int)ceil_div(std::max(nchunks, 1), kWarpsPerCta);
    const size_t smem = sizeof(int32_t) * kWarpsPerCta * a.nr;
    if (a.T > 0) {
        launch_k(count_kernel, dim3(nblk), dim3(32 * kWarpsPerCta), smem, st, a.gidx, a.T, a.K, a.N, a.n_start, a.nr, nchunks, a.whist,
                                                            a.expert_counts, a.err);
        B2_LAUNCH_CHECK();
    }
    launch_k(scan_kernel, dim3(1), dim3(1024), sizeof(int32_t) * a.nr, st, a.whist, nchunks, a.nr, a.expert_counts, a.T, a.wbase,
                                                         a.token_counts, a.cum_token_counts, a.pad_start,
                                                         a.cum_expert_counts, a.expert_order);
    B2_LAUNCH_CHECK();
    if (a.T > 0) {
        launch_k(scatter_kernel, dim3(nblk), dim3(32 * kWarpsPerCta), smem, st, a.gidx, a.T, a.K, a.n_start, a.nr, nchunks, a.wbase,
                                                              a.cum_token_counts, a.pad_start, a.cum_expert_counts,
                                                              a.input_indices, a.output_indices, a.selected_k,
                                                              a.slot_prow, a.prow_src, a.gw, a.prow_w);
        B2_LAUNCH_CHECK();
    }
    launch_k(pad_fill_kernel, dim3(a.nr), dim3(128), 0, st, a.token_counts, a.pad_start, a.nr, a.prow_src, a.prow_w);
    B2_LAUNCH_CHECK();
}

// ---- TBS-blocked diagnostics (export only) ----------------------------------------------

__global__ void partial_count_kernel(const int32_t* __restrict__ gidx, int64_t n, int K, int n_start, int nr, int th,
                                     int tbs, int32_t* __restrict__ partial) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int ln = local_of(gidx[i], n_start, nr);
        if (ln >= 0) atomicAdd(&partial[(int64_t)ln * th + (i / K) / tbs], 1);
    }
}

__global__ void __launch_bounds__(1024) partial_scan_kernel(const int32_t* __restrict__ partial, int64_t n,
                                                            int32_t* __restrict__ partial_cum) {
    __shared__ int wsum[32];
    const int64_t tot = block_scan(
        n, [&](int64_t i) { return partial[i]; }, [&](int64_t i, int64_t v) { partial_cum[i] = (int32_t)v; }, wsum);
    if (threadIdx.x == 0) partial_cum[n] = (int32_t)tot;
}

void launch_partial_counts(const int32_t* gidx, int T, int K, int n_start, int nr, int tbs, int th, int32_t* partial,
                           int32_t* partial_cum, cudaStream_t st) {
    const int64_t np = (int64_t)nr * th;
    B2_CUDA(cudaMemsetAsync(partial, 0, sizeof(int32_t) * (size_t)std::max<int64_t>(np, 1), st));
    const int64_t n = (int64_t)T * K;
    if (n > 0) {
        partial_count_kernel<<<(unsigned)std::min<int64_t>(1184, ceil_div(n, 256)), 256, 0, st>>>(gidx, n, K, n_start,
                                                                                                  nr, th, tbs, partial);
        B2_LAUNCH_CHECK();
    }
    partial_scan_kernel<<<1, 1024, 0, st>>>(partial, np, partial_cum);
    B2_LAUNCH_CHECK();
}

}  // namespace b2
