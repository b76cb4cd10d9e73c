// Expert-parallel dispatch / combine over NVLink peer memory (EP > 1).
//
// The reference gathers every rank's tokens, routing weights and expert ids on every
// rank (allgather, moe.hpp:365-367), computes its experts on the gathered table and
// returns the combined rows with a rank-ordered reducescatter (moe.hpp:378); the
// backward mirrors both (moe.hpp:400, 427-428). Here only the routing TABLE is
// gathered ([S,K] ids + weights, pulled from every rank's symmetric buffer after an NVLink
// flag barrier: the reference's indices_g / weights_g, so counting and index generation
// see exactly the reference's gathered table). Token rows never take a collective:
//   gather   the expert owner PULLS each gathered token that has a local expert once
//            from the source rank's x over NVLink (CUDA IPC mapping) and writes it to
//            every padded row of that token (dedup per destination);
//   combine  the owner combines the token's local slots (weighted, slot order) and PUSHES the
//            partial row into the source rank's slab, row [owner][token] (NVLink stores);
//            after a barrier the source sums the rows of the ranks its token routed to in
//            rank order (the reducescatter's member order, comm.hpp:391-394), locally.
// The backward pulls dout rows the same way and returns dX partial rows by the same push +
// sum; the top-k weight gradients stay in the owners' slabs and are pulled and summed (a
// few KB). No host synchronisation, no staging copies.
#include "b2_common.cuh"
#include "kernels.h"

namespace b2 {

// warp per gathered token gid with local slots: pull its row once, write all its rows
template <typename T>
__global__ void ep_gather_pull_kernel(const T* const* __restrict__ peer_src, int S, int T_tot, int H,
                                      const int32_t* __restrict__ cec, const int32_t* __restrict__ slot_prow,
                                      T* __restrict__ out) {
    pdl_wait();
    pdl_launch();
    const int lane = threadIdx.x % 32;
    const int nw = gridDim.x * blockDim.x / 32;
    for (int gid = (blockIdx.x * blockDim.x + threadIdx.x) / 32; gid < T_tot; gid += nw) {
        const int j0 = cec[gid], j1 = cec[gid + 1];
        if (j0 == j1) continue;
        const T* src = peer_src[gid / S] + (int64_t)(gid % S) * H;
        if (((int64_t)H * sizeof(T)) % 16 == 0) {
            // up to 8 x 16 B of the remote row in flight per lane (a 4 KB row per warp), then
            // the local copies: NVLink latency is hidden by bytes in flight, not by occupancy
            constexpr int B = 8;
            const int nv = (int)((int64_t)H * sizeof(T) / 16);
            for (int v0 = 0; v0 < nv; v0 += 32 * B) {
                int4 val[B];
#pragma unroll
                for (int b = 0; b < B; ++b) {
                    const int v = v0 + lane + 32 * b;
                    if (v < nv) val[b] = reinterpret_cast<const int4*>(src)[v];
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
        } else {
            for (int c = lane; c < H; c += 32) {
                const T val = src[c];
                for (int j = j0; j < j1; ++j) out[(int64_t)slot_prow[j] * H + c] = val;
            }
        }
    }
}

// the owner's (weighted) sum of a gathered token's local slot rows, in slot (k) order, into
// its own slab row [gid] or pushed into the source's slab row [me][token];
// (256, 4): 32 resident warps per SM instead of 24 for these latency-bound row loops (EP 4
// 5.58-5.59 -> 5.55-5.56 ms per step, EP 2 unchanged)
template <typename T>
__global__ void __launch_bounds__(256, 4) ep_combine_slots_kernel(const T* __restrict__ y, const int32_t* __restrict__ slot_prow,
                                           const int32_t* __restrict__ selected_k, const int32_t* __restrict__ cec,
                                           const float* __restrict__ gw, int K, int T_tot, int H,
                                           T* __restrict__ own_slab, T* const* __restrict__ push_slab, int S,
                                           int me) {
    pdl_wait();
    pdl_launch();
    constexpr int V = 16 / sizeof(T);
    const int lane = threadIdx.x % 32;
    const int nw = gridDim.x * blockDim.x / 32;
    const int nv = H / V;
    for (int gid = (blockIdx.x * blockDim.x + threadIdx.x) / 32; gid < T_tot; gid += nw) {
        const int j0 = cec[gid], j1 = cec[gid + 1];
        if (j0 == j1) continue;
        // push: straight into the source rank's slab, row [me][token] (NVLink stores)
        T* dst = push_slab ? push_slab[gid / S] + ((int64_t)me * S + gid % S) * H : own_slab + (int64_t)gid * H;
        // all local slot rows of a column block are loaded together (<= 8 in flight)
        constexpr int MAXJ = 8;
        for (int v = lane; v < nv; v += 32) {
            float acc[V];
#pragma unroll
            for (int q = 0; q < V; ++q) acc[q] = 0.f;
            for (int jb = j0; jb < j1; jb += MAXJ) {
                const int nj = min(MAXJ, j1 - jb);
                int4 raw[MAXJ];
#pragma unroll
                for (int q = 0; q < MAXJ; ++q)
                    if (q < nj) raw[q] = __ldg(reinterpret_cast<const int4*>(y + (int64_t)slot_prow[jb + q] * H) + v);
#pragma unroll
                for (int q = 0; q < MAXJ; ++q) {
                    if (q >= nj) break;
                    float f[V];
                    if constexpr (sizeof(T) == 4) {
                        f[0] = __int_as_float(raw[q].x);
                        f[1] = __int_as_float(raw[q].y);
                        f[2] = __int_as_float(raw[q].z);
                        f[3] = __int_as_float(raw[q].w);
                    } else {
                        const uint32_t w[4] = {(uint32_t)raw[q].x, (uint32_t)raw[q].y, (uint32_t)raw[q].z,
                                               (uint32_t)raw[q].w};
#pragma unroll
                        for (int z = 0; z < 4; ++z) {
                            f[2 * z] = __uint_as_float(w[z] << 16);
                            f[2 * z + 1] = __uint_as_float(w[z] & 0xFFFF0000u);
                        }
                    }
                    const float wv = gw ? gw[(int64_t)gid * K + selected_k[jb + q]] : 1.f;
#pragma unroll
                    for (int z = 0; z < V; ++z)
                        acc[z] = gw ? __fadd_rn(acc[z], __fmul_rn(wv, f[z])) : __fadd_rn(acc[z], f[z]);
                }
            }
            int4 o;
            if constexpr (sizeof(T) == 4) {
                o = make_int4(__float_as_int(acc[0]), __float_as_int(acc[1]), __float_as_int(acc[2]),
                              __float_as_int(acc[3]));
            } else {
                uint32_t w[4];
#pragma unroll
                for (int z = 0; z < 4; ++z) {
                    __nv_bfloat162 b = __floats2bfloat162_rn(acc[2 * z], acc[2 * z + 1]);
                    w[z] = *reinterpret_cast<uint32_t*>(&b);
                }
                o = make_int4((int)w[0], (int)w[1], (int)w[2], (int)w[3]);
            }
            reinterpret_cast<int4*>(dst)[v] = o;
        }
    }
}

// out[t] = sum over the ranks r (in order) that token t routes to of owner r's partial row:
// pushed, row [r * S + t] of this rank's own slab; pulled, row [me * S + t] of r's slab over
// NVLink (both written before the barrier) — the reducescatter of moe.hpp:378 / 427-428 in
// member order, with up to 8 owners' 16-byte vectors in flight per lane
template <typename T>
__device__ __forceinline__ void ep_pull_sum_token(const T* const* __restrict__ peer_slab,
                                                  const int32_t* __restrict__ gi_local, int S, int K, int E, int NR,
                                                  int W, int me, T* __restrict__ out, int t, int lane, bool pushed) {
    unsigned mask = 0;
    for (int k = 0; k < K; ++k) mask |= 1u << (gi_local[(int64_t)t * K + k] / NR);
    // pulled: owner r's own slab, row [me][t]; pushed: this rank's slab, row [r][t]
    auto src = [&](int r) -> const T* {
        return pushed ? peer_slab[me] + ((int64_t)r * S + t) * W : peer_slab[r] + ((int64_t)me * S + t) * W;
    };
    if (((int64_t)W * sizeof(T)) % 16 == 0) {
        constexpr int V = 16 / sizeof(T), MAXR = 8;
        for (int v = lane; v < W / V; v += 32) {
            float acc[V];
            bool any = false;
            for (int r0 = 0; r0 < E; r0 += MAXR) {
                int4 raw[MAXR];
#pragma unroll
                for (int q = 0; q < MAXR; ++q)
                    if (r0 + q < E && (mask >> (r0 + q) & 1u))
                        raw[q] = __ldcv(reinterpret_cast<const int4*>(src(r0 + q)) + v);
#pragma unroll
                for (int q = 0; q < MAXR; ++q) {
                    if (!(r0 + q < E && (mask >> (r0 + q) & 1u))) continue;
                    float f[V];
                    if constexpr (sizeof(T) == 4) {
                        f[0] = __int_as_float(raw[q].x);
                        f[1] = __int_as_float(raw[q].y);
                        f[2] = __int_as_float(raw[q].z);
                        f[3] = __int_as_float(raw[q].w);
                    } else {
                        const uint32_t w[4] = {(uint32_t)raw[q].x, (uint32_t)raw[q].y, (uint32_t)raw[q].z,
                                               (uint32_t)raw[q].w};
#pragma unroll
                        for (int z = 0; z < 4; ++z) {
                            f[2 * z] = __uint_as_float(w[z] << 16);
                            f[2 * z + 1] = __uint_as_float(w[z] & 0xFFFF0000u);
                        }
                    }
#pragma unroll
                    for (int z = 0; z < V; ++z) acc[z] = any ? __fadd_rn(acc[z], f[z]) : f[z];
                    any = true;
                }
            }
            if (!any)
                for (int z = 0; z < V; ++z) acc[z] = 0.f;
            int4 o;
            if constexpr (sizeof(T) == 4) {
                o = make_int4(__float_as_int(acc[0]), __float_as_int(acc[1]), __float_as_int(acc[2]),
                              __float_as_int(acc[3]));
            } else {
                uint32_t w[4];
#pragma unroll
                for (int z = 0; z < 4; ++z) {
                    __nv_bfloat162 b = __floats2bfloat162_rn(acc[2 * z], acc[2 * z + 1]);
                    w[z] = *reinterpret_cast<uint32_t*>(&b);
                }
                o = make_int4((int)w[0], (int)w[1], (int)w[2], (int)w[3]);
            }
            reinterpret_cast<int4*>(out + (int64_t)t * W)[v] = o;
        }
    } else {
        for (int c = lane; c < W; c += 32) {
            float acc = 0.f;
            bool any = false;
            for (int r = 0; r < E; ++r) {
                if (!(mask >> r & 1u)) continue;
                const float v = Elem<T>::to_f(__ldcv(src(r) + c));
                acc = any ? __fadd_rn(acc, v) : v;
                any = true;
            }
            out[(int64_t)t * W + c] = Elem<T>::from_f(acc);
        }
    }
}

template <typename T>
__global__ void __launch_bounds__(256, 4) ep_pull_sum_kernel(const T* const* __restrict__ peer_slab, const int32_t* __restrict__ gi_local,
                                   int S, int K, int E, int NR, int W, int me, T* __restrict__ out, int pushed) {
    pdl_wait();
    pdl_launch();
    const int lane = threadIdx.x % 32, nw = gridDim.x * blockDim.x / 32;
    for (int t = (blockIdx.x * blockDim.x + threadIdx.x) / 32; t < S; t += nw)  // grid-stride: any grid size
        ep_pull_sum_token<T>(peer_slab, gi_local, S, K, E, NR, W, me, out, t, lane, pushed != 0);
}

// NVLink flag barrier over the EP group: every rank bumps its slot in every peer's flag
// array (system-scope release), then waits until all of its own slots reach the epoch it
// expects (acquire). Epochs live on the device (graph-replay safe); every rank calls the
// barriers in the same order, so the counts agree. Bounded spin: traps after ~20 s.
__global__ void ep_flag_barrier_kernel(int* const* __restrict__ peer_flags, int* __restrict__ own_flags,
                                       int* __restrict__ epoch, int E, int me) {
    pdl_wait();
    pdl_launch();
    const int p = threadIdx.x;
    __shared__ int target;
    if (p == 0) target = *epoch + 1;
    __syncthreads();
    __threadfence_system();  // this rank's earlier stores (incl. peer memory) before the signal
    if (p < E) atomicAdd_system(peer_flags[p] + me, 1);
    if (p < E) {
        uint64_t t0 = 0;
        unsigned spins = 0;
        while (atomicAdd_system(own_flags + p, 0) < target) {
            if ((++spins & 0xFFFu) == 0) {
                uint64_t now;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
                if (t0 == 0) t0 = now;
                else if (now - t0 > 20000000000ull) {
                    printf("b2 ep barrier stuck: rank %d waits on %d (epoch %d)\n", me, p, target);
                    __trap();
                }
            }
        }
    }
    __syncthreads();
    __threadfence_system();
    if (p == 0) *epoch = target;
}

void launch_ep_flag_barrier(int* const* peer_flags, int* own_flags, int* epoch, int E, int me, cudaStream_t st) {
    check(E <= 1024, "ep barrier: group too large");
    launch_k(ep_flag_barrier_kernel, dim3(1), dim3(std::max(32, (E + 31) / 32 * 32)), 0, st, peer_flags, own_flags, epoch, E, me);
    B2_LAUNCH_CHECK();
}

// the routing tables of all EP ranks (the reference's allgathered indices_g / weights_g,
// moe.hpp:366-367), pulled from the peers' symmetric buffers after a barrier
__global__ void ep_table_pull_kernel(const int32_t* const* __restrict__ peer_ids,
                                     const float* const* __restrict__ peer_w, int64_t n, int E,
                                     int32_t* __restrict__ ids_all, float* __restrict__ w_all) {
    pdl_wait();
    pdl_launch();
    const int64_t total = n * E;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int r = (int)(i / n);
        const int64_t j = i % n;
        ids_all[i] = __ldcv(peer_ids[r] + j);
        w_all[i] = __ldcv(peer_w[r] + j);
    }
}

void launch_ep_table_pull(const int32_t* const* peer_ids, const float* const* peer_w, int64_t n, int E,
                          int32_t* ids_all, float* w_all, cudaStream_t st) {
    if (n <= 0) return;
    launch_k(ep_table_pull_kernel, dim3((unsigned)std::min<int64_t>(1184, ceil_div(n * E, 256))), dim3(256), 0, st, peer_ids, peer_w, n, E,
                                                                                                ids_all, w_all);
    B2_LAUNCH_CHECK();
}

static unsigned ep_grid(int64_t warps) { return (unsigned)std::max<int64_t>(1, std::min<int64_t>(148 * 16, ceil_div(warps, 8))); }

template <typename T>
void launch_ep_gather_pull(const T* const* peer_src, int S, int T_tot, int H, const int32_t* cec,
                           const int32_t* slot_prow, T* out, cudaStream_t st) {
    if (T_tot <= 0) return;
    launch_k(ep_gather_pull_kernel<T>, dim3(ep_grid(T_tot)), dim3(256), 0, st, peer_src, S, T_tot, H, cec, slot_prow, out);
    B2_LAUNCH_CHECK();
}

template <typename T>
void launch_ep_combine_local(const T* y, const int32_t* slot_prow, const int32_t* selected_k, const int32_t* cec,
                             const float* gw, int K, int S, int T_tot, int H, T* own_slab, cudaStream_t st,
                             int max_blocks, T* const* push_slab, int me) {
    if (T_tot <= 0) return;
    check(((int64_t)H * sizeof(T)) % 16 == 0, "ep combine: rows must be 16-byte multiples");
    const unsigned grid = max_blocks > 0 ? std::min<unsigned>(ep_grid(T_tot), (unsigned)max_blocks) : ep_grid(T_tot);
    launch_k(ep_combine_slots_kernel<T>, dim3(grid), dim3(256), 0, st, y, slot_prow, selected_k, cec, gw, K, T_tot, H,
             own_slab, push_slab, S, me);
    B2_LAUNCH_CHECK();
}

template <typename T>
void launch_ep_pull_sum(const T* const* peer_slab, const int32_t* gi_local, int S, int K, int E, int NR, int W, int me,
                        T* out, cudaStream_t st, int max_blocks, bool pushed) {
    if (S <= 0) return;
    const unsigned full = (unsigned)ceil_div(S, 8);
    launch_k(ep_pull_sum_kernel<T>, dim3(max_blocks > 0 ? std::min<unsigned>(full, (unsigned)max_blocks) : full), dim3(256), 0, st, peer_slab, gi_local, S, K, E, NR, W, me, out, pushed ? 1 : 0);
    B2_LAUNCH_CHECK();
}

#define B2_EP_INST(T)                                                                                             \
    template void launch_ep_gather_pull<T>(const T* const*, int, int, int, const int32_t*, const int32_t*, T*,    \
                                           cudaStream_t);                                                         \
    template void launch_ep_combine_local<T>(const T*, const int32_t*, const int32_t*, const int32_t*, const float*, \
                                             int, int, int, int, T*, cudaStream_t, int, T* const*, int);        \
    template void launch_ep_pull_sum<T>(const T* const*, const int32_t*, int, int, int, int, int, int, T*,        \
                                        cudaStream_t, int, bool);
B2_EP_INST(float)
B2_EP_INST(__nv_bfloat16)
#undef B2_EP_INST

}  // namespace b2
