// Token counting and index generation (Algorithm 1 stages 2-3) on the gathered
// routing table, bit-exact with the reference.
//
// Reference: count_tokens (include/optimus/moe.hpp:122-164) and generate_indices
// (moe.hpp:167-197). The reference's result is a STABLE sort of the local
// selections by expert, in (token, k) order within an expert, independent of the
// token-block size (test_moe.cpp:130-207). Here:
//   1. one warp per 64-token chunk builds a shared-memory histogram of its local
//      selections (counts are order-free, so smem atomics are deterministic);
//   2. one CTA scans the histograms in (expert-major, chunk-minor) order, giving
//      each (expert, chunk) its first row; it also scans per-token counts
//      (cum_expert_counts), the TBS-blocked diagnostics (partial_cum) and the
//      128-row padded group starts used by the GEMMs;
//   3. each warp re-walks its chunk in (t, k) order in 32-entry batches and ranks
//      equal experts with __match_any_sync plus a per-expert carry, so the row of
//      every selection equals the reference's counter(ln, tid)++.
#include "b2_common.cuh"
#include "kernels.h"

namespace b2 {

constexpr int kChunk = 64;           // tokens per warp chunk
constexpr int kWarpsPerCta = 4;

__device__ __forceinline__ int local_of(int e, int n_start, int nr) {
    return (e >= n_start && e < n_start + nr) ? e - n_start : -1;
}

// 1. histograms + per-token local counts + TBS-blocked counts
__global__ void count_kernel(const int32_t* __restrict__ gidx, int T, int K, int N, int n_start, int nr, int tbs,
                             int th, int32_t* __restrict__ whist /*[nchunks][nr]*/,
                             int32_t* __restrict__ expert_counts, int32_t* __restrict__ partial_counts,
                             int32_t* __restrict__ err) {
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
            const int t = t0 + f / K;
            const int e = gidx[(int64_t)t0 * K + f];
            if (e < 0 || e >= N) {
                atomicExch(err, 1);
                continue;
            }
            const int ln = local_of(e, n_start, nr);
            if (ln >= 0) {
                atomicAdd(&hist[ln], 1);
                atomicAdd(&partial_counts[(int64_t)ln * th + t / tbs], 1);
            }
        }
        for (int t = t0 + lane; t < t1; t += 32) {
            int c = 0;
            for (int k = 0; k < K; ++k) c += local_of(gidx[(int64_t)t * K + k], n_start, nr) >= 0;
            expert_counts[t] = c;
        }
    }
    __syncwarp();
    const int nchunks = (int)ceil_div(T, kChunk);
    if (chunk < nchunks)
        for (int i = lane; i < nr; i += 32) whist[(int64_t)chunk * nr + i] = hist[i];
}

// block-wide exclusive scan of n ints read through `get(i)`, results through `put(i, v)`;
// returns the total. Each thread owns one contiguous segment (fixed order).
template <class Get, class Put>
__device__ int64_t block_exclusive_scan(int64_t n, Get get, Put put, int64_t* sh_partials) {
    const int tid = threadIdx.x, nt = blockDim.x;
    const int64_t seg = ceil_div(n, nt);
    const int64_t b = min(n, (int64_t)tid * seg), e = min(n, b + seg);
    int64_t s = 0;
    for (int64_t i = b; i < e; ++i) s += get(i);
    sh_partials[tid] = s;
    __syncthreads();
    if (tid == 0) {
        int64_t acc = 0;
        for (int i = 0; i < nt; ++i) {
            const int64_t v = sh_partials[i];
            sh_partials[i] = acc;
            acc += v;
        }
        sh_partials[nt] = acc;
    }
    __syncthreads();
    int64_t acc = sh_partials[tid];
    for (int64_t i = b; i < e; ++i) {
        const int64_t v = get(i);
        put(i, acc);
        acc += v;
    }
    const int64_t total = sh_partials[nt];
    __syncthreads();
    return total;
}

// 2. all scans, one CTA of 1024 threads
__global__ void __launch_bounds__(1024) scan_kernel(const int32_t* __restrict__ whist, int nchunks, int nr,
                                                    const int32_t* __restrict__ expert_counts, int T,
                                                    const int32_t* __restrict__ partial_counts, int th,
                                                    int32_t* __restrict__ wbase /*[nchunks][nr]*/,
                                                    int32_t* __restrict__ token_counts,
                                                    int32_t* __restrict__ cum_token_counts,
                                                    int32_t* __restrict__ pad_start,
                                                    int32_t* __restrict__ cum_expert_counts,
                                                    int32_t* __restrict__ partial_cum) {
    __shared__ int64_t part[1025];
    // (expert-major, chunk-minor) scan of the chunk histograms
    const int64_t n1 = (int64_t)nr * nchunks;
    const int64_t rt = block_exclusive_scan(
        n1, [&](int64_t i) { return (int64_t)whist[(i % nchunks) * nr + i / nchunks]; },
        [&](int64_t i, int64_t v) { wbase[(i % nchunks) * nr + i / nchunks] = (int32_t)v; }, part);
    // expert totals, group boundaries and padded starts (thread 0: nr is small)
    if (threadIdx.x == 0) {
        // cum_token_counts[ln] = partial_cum[ln * TH] in the reference (moe.hpp:156-158):
        // here the scan value at (ln, chunk 0)
        int64_t pacc = 0;
        for (int ln = 0; ln < nr; ++ln) {
            const int64_t b = nchunks ? wbase[ln] : 0;
            const int64_t e = (ln + 1 < nr) ? (nchunks ? wbase[ln + 1] : 0) : rt;
            token_counts[ln] = (int32_t)(e - b);
            cum_token_counts[ln] = (int32_t)b;
            pad_start[ln] = (int32_t)pacc;
            pacc += round_up(e - b, kRowAlign);
        }
        cum_token_counts[nr] = (int32_t)rt;
        pad_start[nr] = (int32_t)pacc;
    }
    __syncthreads();
    const int64_t tot_e = block_exclusive_scan(
        T, [&](int64_t i) { return (int64_t)expert_counts[i]; },
        [&](int64_t i, int64_t v) { cum_expert_counts[i] = (int32_t)v; }, part);
    if (threadIdx.x == 0) cum_expert_counts[T] = (int32_t)tot_e;
    const int64_t n3 = (int64_t)nr * th;
    const int64_t tot_p = block_exclusive_scan(
        n3, [&](int64_t i) { return (int64_t)partial_counts[i]; },
        [&](int64_t i, int64_t v) { partial_cum[i] = (int32_t)v; }, part);
    if (threadIdx.x == 0) partial_cum[n3] = (int32_t)tot_p;
}

// 3. stable scatter
__global__ void scatter_kernel(const int32_t* __restrict__ gidx, int T, int K, int n_start, int nr,
                               const int32_t* __restrict__ wbase, const int32_t* __restrict__ cum_token_counts,
                               const int32_t* __restrict__ pad_start, const int32_t* __restrict__ cum_expert_counts,
                               int32_t* __restrict__ input_indices, int32_t* __restrict__ output_indices,
                               int32_t* __restrict__ selected_k, int32_t* __restrict__ slot_prow,
                               int32_t* __restrict__ prow_src) {
    extern __shared__ int32_t sh[];  // carry [kWarpsPerCta][nr]
    const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int chunk = blockIdx.x * kWarpsPerCta + w;
    const int t0 = chunk * kChunk;
    if (t0 >= T) return;
    int32_t* carry = sh + w * nr;
    for (int i = lane; i < nr; i += 32) carry[i] = wbase[(int64_t)chunk * nr + i];
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
        int row = 0;
        if (ln >= 0) row = carry[ln] + __popc(peers & lt);
        __syncwarp();
        if (ln >= 0 && (peers & lt) == 0) carry[ln] += __popc(peers);  // group leader
        __syncwarp();
        if (ln >= 0) {
            int before = 0;  // local selections of token t with k' < k
            for (int kk = 0; kk < k; ++kk) before += local_of(gidx[(int64_t)t * K + kk], n_start, nr) >= 0;
            const int pos = cum_expert_counts[t] + before;
            const int prow = pad_start[ln] + (row - cum_token_counts[ln]);
            input_indices[row] = t;
            output_indices[pos] = row;
            selected_k[pos] = k;
            slot_prow[pos] = prow;
            prow_src[prow] = t;
        }
    }
}

// pad rows of each expert group read as zero tokens
__global__ void pad_fill_kernel(const int32_t* __restrict__ token_counts, const int32_t* __restrict__ pad_start,
                                int nr, int32_t* __restrict__ prow_src) {
    const int ln = blockIdx.x;
    const int b = pad_start[ln] + token_counts[ln], e = pad_start[ln + 1];
    for (int r = b + threadIdx.x; r < e; r += blockDim.x) prow_src[r] = -1;
}

void launch_routing_index(const RoutingIndexArgs& a, cudaStream_t st) {
    const int nchunks = (int)ceil_div(a.T, kChunk);
    const int nblk = (int)ceil_div(std::max(nchunks, 1), kWarpsPerCta);
    const size_t smem = sizeof(int32_t) * kWarpsPerCta * a.nr;
    B2_CUDA(cudaMemsetAsync(a.partial_counts, 0, sizeof(int32_t) * (size_t)a.nr * a.th, st));
    if (a.T > 0) {
        count_kernel<<<nblk, 32 * kWarpsPerCta, smem, st>>>(a.gidx, a.T, a.K, a.N, a.n_start, a.nr, a.tbs, a.th,
                                                            a.whist, a.expert_counts, a.partial_counts, a.err);
        B2_LAUNCH_CHECK();
    }
    scan_kernel<<<1, 1024, 0, st>>>(a.whist, nchunks, a.nr, a.expert_counts, a.T, a.partial_counts, a.th, a.wbase,
                                    a.token_counts, a.cum_token_counts, a.pad_start, a.cum_expert_counts,
                                    a.partial_cum);
    B2_LAUNCH_CHECK();
    if (a.T > 0) {
        scatter_kernel<<<nblk, 32 * kWarpsPerCta, smem, st>>>(a.gidx, a.T, a.K, a.n_start, a.nr, a.wbase,
                                                              a.cum_token_counts, a.pad_start, a.cum_expert_counts,
                                                              a.input_indices, a.output_indices, a.selected_k,
                                                              a.slot_prow, a.prow_src);
        B2_LAUNCH_CHECK();
    }
    pad_fill_kernel<<<a.nr, 128, 0, st>>>(a.token_counts, a.pad_start, a.nr, a.prow_src);
    B2_LAUNCH_CHECK();
}

}  // namespace b2
