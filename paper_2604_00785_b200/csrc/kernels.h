// Kernel launchers of the B200 MoE expert path (all asynchronous on `st`).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace b2 {

// ---- router (route.cu) ----
template <typename T>
void launch_router_logits(const T* x, const T* w, float* logits, int S, int H, int N, cudaStream_t st);
void launch_softmax_topk(const float* logits, float* probs, float* topw, int32_t* topi, int S, int N, int K,
                         bool normalize, cudaStream_t st);
void launch_fur_route(float* w, int32_t* idx, int S, int N, int K, cudaStream_t st);
// partial: [ceil(S/128), N] scratch; ctr: one int32, zero before the first call (left zero)
void launch_aux_stats(const float* probs, int S, int N, const int32_t* gidx, int64_t n_gidx, float* partial,
                      int32_t* ctr, float* mean_probs, int32_t* sel, cudaStream_t st);
// dl_bf16 (optional): bf16(dlogits) for the tensor-core router GEMMs; dl_lo (optional):
// bf16(dlogits - dl_bf16), the low half of a two-term split (RouterDx)
void launch_router_dlogits(const float* probs, const float* wgrad, const int32_t* topi, const float* topw,
                           const float* aux_grad, float* dlogits, void* dl_bf16, void* dl_lo, int S, int N, int K,
                           bool normalize, bool fur, cudaStream_t st);
void launch_aux_probs_grad(const int32_t* sel, float* out, int S, int N, double coeff, double total,
                           cudaStream_t st);
// dWr = x^T dlogits with a deterministic split over S; part holds max_splits*H*N floats
template <typename T>
void launch_router_dw(const T* x, const float* dlogits, T* dw, float* part, int max_splits, int S, int H, int N,
                      cudaStream_t st);

constexpr int kRouterDwMaxSplits = 32;

// ---- counting / index generation (index.cu) ----
struct RoutingIndexArgs {
    const int32_t* gidx;  // [T, K] gathered expert ids
    int T, K, N, n_start, nr;
    int32_t* whist;              // [nr, ceil(T/64)]
    int32_t* wbase;              // [nr, ceil(T/64)]
    int32_t* expert_counts;      // [T]
    int32_t* cum_expert_counts;  // [T+1]
    int32_t* token_counts;       // [nr]
    int32_t* cum_token_counts;   // [nr+1]
    int32_t* pad_start;          // [nr+1]
    int32_t* input_indices;      // [T*K] compact row -> token
    int32_t* output_indices;     // [T*K] token-major slot -> compact row
    int32_t* selected_k;         // [T*K]
    int32_t* slot_prow;          // [T*K] token-major slot -> padded row
    int32_t* prow_src;           // [pmax] padded row -> token (-1 pad)
    const float* gw;             // [T, K] dispatch weights (with prow_w)
    float* prow_w;               // [pmax] padded row -> its routing weight (0 pad); nullptr: not needed
    int32_t* err;                // expert id out of range flag
    int32_t* expert_order;       // [nr] experts by descending row count (wgrad tile order); nullptr: none
};
void launch_routing_index(const RoutingIndexArgs& a, cudaStream_t st);
// TBS-blocked diagnostics partial_token_counts [nr*th] / partial_cum [nr*th+1] (moe.hpp:148-158)
void launch_partial_counts(const int32_t* gidx, int T, int K, int n_start, int nr, int tbs, int th, int32_t* partial,
                           int32_t* partial_cum, cudaStream_t st);

// ---- permute / combine / element-wise (permute.cu) ----
template <typename T>
void launch_gather_rows(const T* x, const int32_t* prow_src, const int32_t* p_total, T* out, int H, int64_t pmax,
                        cudaStream_t st);
template <typename T>
void launch_zero_pad_rows(T* buf, const int32_t* prow_src, const int32_t* p_total, int W, int64_t pmax,
                          cudaStream_t st);
// the gather token-major (each x row read once, written to its padded rows slot_prow[cec[t]..]),
// pad rows zeroed in the same launch
template <typename T>
void launch_gather_tokens(const T* x, const int32_t* cec, const int32_t* slot_prow, int T_tok,
                          const int32_t* prow_src, const int32_t* p_total, T* out, int H, int64_t pmax,
                          cudaStream_t st);
template <typename T>
void launch_combine(const T* y, const int32_t* slot_prow, const int32_t* selected_k, const int32_t* cec,
                    const float* gw, T* out, int T_tok, int H, int K, cudaStream_t st);
template <typename T>
void launch_out_reduction_bwd(const T* dout, const T* const* peer_dout, int s_local, const T* y,
                              const int32_t* slot_prow, const int32_t* selected_k, const int32_t* cec, const float* gw,
                              T* dy, float* wgrad, int T_tok, int H, int K, cudaStream_t st);
// bf16 path: wgrad[t, k] from the dgrad epilogue's np partial dots per padded row
void launch_wgrad_from_parts(const float* part, int np, const int32_t* slot_prow, const int32_t* selected_k,
                             const int32_t* cec, float* wgrad, int T_tok, int K, cudaStream_t st);
template <typename T>
void launch_dx_finalize(const T* src, bool from_slots, const int32_t* slot_prow, const int32_t* cec, const float* dl,
                        const T* wr, T* dx, int S, int H, int N, cudaStream_t st);
template <typename T>
void launch_swiglu_fwd(const T* g, const T* u, T* h, const int32_t* p_total, int I, int64_t pmax, cudaStream_t st);
template <typename T>
void launch_swiglu_bwd(const T* g, const T* u, const T* dh, T* dgu, const int32_t* p_total, int I, int64_t pmax,
                       cudaStream_t st);

// ---- expert-parallel dispatch / combine over NVLink peer memory (ep_dispatch.cu) ----
template <typename T>
void launch_ep_gather_pull(const T* const* peer_src, int S, int T_tot, int H, const int32_t* cec,
                           const int32_t* slot_prow, T* out, cudaStream_t st);
// owner side of the combine: the token's (weighted) partial row into the owner's OWN slab row
// [gid] (sources pull them after a barrier), or with push_slab (the E slab pointers) straight
// into the source rank's slab row [me][token] (the sources then sum locally, pushed = true)
template <typename T>
void launch_ep_combine_local(const T* y, const int32_t* slot_prow, const int32_t* selected_k, const int32_t* cec,
                             const float* gw, int K, int S, int T_tot, int H, T* own_slab, cudaStream_t st,
                             int max_blocks = 0, T* const* push_slab = nullptr, int me = 0);
// out[t] = sum over t's owner ranks (in rank order) of peer_slab[r][(me*S + t)*W ..]
template <typename T>
// max_blocks > 0 caps the grid (a side-stream launch that must stay inside its reserved SMs)
void launch_ep_pull_sum(const T* const* peer_slab, const int32_t* gi_local, int S, int K, int E, int NR, int W, int me,
                        T* out, cudaStream_t st, int max_blocks = 0, bool pushed = false);
// [E][n] routing tables gathered from the peers' symmetric buffers
void launch_ep_table_pull(const int32_t* const* peer_ids, const float* const* peer_w, int64_t n, int E,
                          int32_t* ids_all, float* w_all, cudaStream_t st);
// all-ranks barrier over NVLink peer memory (flag counters in the symmetric buffer)
void launch_ep_flag_barrier(int* const* peer_flags, int* own_flags, int* epoch, int E, int me, cudaStream_t st);
// ---- SIMT grouped GEMM (simt_gemm.cu) ----
struct SimtGemmArgs {
    const void* A;
    const void* B;
    void* D;
    int64_t lda_m, lda_k, a_gs;
    int64_t ldb_k, ldb_n, b_gs;
    int64_t ldd_m, ldd_n, d_gs;
    const int32_t* group_start;  // [groups+1]
    int groups;
    int by_k;
    int64_t M_lim;  // by_k: M; by_m: row capacity
    int N, K;       // K used by by_m
    float scale;
    int accumulate;
};
template <typename T>
void launch_simt_grouped_gemm(const SimtGemmArgs& a, int64_t m_extent, cudaStream_t st);

// ---- tcgen05 grouped GEMM (gemm_sm100.cu) ----
enum class GemmKind : int {
    FwdGateUp = 0,   // [G|U] = X · [Wg|Wu], epilogue: G, U, H = silu(G)·U
    FwdDown = 1,     // Y = H · Wd
    BwdDownDgrad = 2,// dH = dY · Wdᵀ, epilogue: SwiGLU backward -> dGU = [dG | dU]
    BwdDx = 3,       // dX = [dG|dU] · [Wg|Wu]ᵀ   (K = 2I)
    WgradDown = 4,   // dWd[e] = Hᵀ · dY  over the rows of e
    WgradGateUp = 5, // [dWg|dWu][e] = Xᵀ · [dG|dU]
    RouterDx = 6,    // dx = base + dlogits · Wrᵀ   (M = S, K = 2 x N experts: the hi + lo dlogits split)
    RouterDw = 7,    // dWr partials [split][H][N] = x[rows of split]ᵀ · dlogits (split-K over S)
};
struct Sm100GemmArgs {
    GemmKind kind;
    int H, I, nr;              // layer dims, local experts
    int64_t pmax;              // padded row capacity
    const int32_t* pad_start;  // [nr+1] device
    const int32_t* counts;     // [nr] device rows per expert (wgrad kinds)
    // operands (bf16), meaning depends on kind
    const void* x;      // mlp_in [P, H]
    const void* wg;     // [nr, H, I]
    const void* wu;     // [nr, H, I]
    const void* wd;     // [nr, I, H]
    const void* g;      // [P, I]
    const void* u;      // [P, I]
    const void* h;      // [P, I]
    const void* dy;     // [P, H]
    const void* dgu;    // [P, 2I]
    void* out0;         // kind-specific outputs
    void* out1;
    void* out2;
    float scale;        // wgrad: 1/EP
    // bf16 layer (weighted-H scheme): row_w [P] = each padded row's routing weight. FwdGateUp
    // stores H' = w * silu(G) * U; BwdDownDgrad takes the UNweighted dout rows as dY, scales its
    // accumulator by w and leaves the top-k weight-gradient partial dots acc . silu(G) * U in
    // wpart [P, I / 64] (null row_w: plain semantics, dY already weighted)
    const float* row_w;
    float* wpart;
    const int32_t* expert_order;  // wgrad kinds: expert of the i-th group of tiles (null: i)
    int num_sms;
    // router kinds
    int S, N;                    // local tokens, experts
    const void* wr;              // router weight [H, N] bf16
    const void* dl;              // dlogits [S, N] bf16 (RouterDx: the high half of the split)
    const void* dl_lo;           // RouterDx: bf16(dlogits - dl) [S, N]
    const void* src;             // RouterDx: base rows [S, H] (the token's summed expert-gradient rows)
    float* part;                 // RouterDw: fp32 partials [nsplit][H][N]
    int nsplit_out;              // RouterDw: number of S splits used (set by the launcher)
    int max_ctas;                // > 0: cap the persistent grid (SMs left to concurrent comm kernels)
};
void launch_sm100_gemm(const Sm100GemmArgs& a, cudaStream_t st);
// number of S splits the RouterDw kind uses (its partial buffer holds splits*H*N floats)
int router_dw_splits(int64_t S, int64_t H, int num_sms);
// sums RouterDw partials in split order into dW (T = bf16)
void launch_router_dw_reduce_bf16(const float* part, void* dw, int nsplit, int64_t n, cudaStream_t st);
bool sm100_available();

// ---- optimizer (adamw.cu) ----
struct AdamWKernelArgs {
    float* master;
    float* m;
    float* v;
    const void* grad;   // owned slice, grad_dtype
    void* weight_out;   // owned slice of the weight, weight_dtype
    int64_t n;
    int grad_dtype, weight_dtype;
    double lr, beta1, beta2, eps, weight_decay, bc1, bc2;
    double grad_scale;  // 1/g (the reduce-scatter mean) applied as (float)(g * (float)scale)
    double clip;        // clip scale (1.0: off)
    int round_bf16;
};
void launch_adamw(const AdamWKernelArgs& a, cudaStream_t st);
// norm_sq: device fp64 global sum of squares; the clip scale is derived on the device
void launch_adamw_full(const AdamWKernelArgs& a, const double* norm_sq, double clip_norm, int clip_active,
                       cudaStream_t st);
// *acc (=|+=) sum of squares of (float)(g * scale); partials holds >= nparts doubles
void launch_sumsq_acc(const void* g, int dtype, int64_t n, float scale, double* partials, int nparts, double* acc,
                      bool init, cudaStream_t st);
void launch_scale_inplace(void* buf, int dtype, int64_t n, float scale, cudaStream_t st);
// sum of squares of an fp32/bf16 slice (after the 1/g scale), fp64 partials
void launch_sumsq(const void* g, int dtype, int64_t n, double scale, double* partials, int nparts, cudaStream_t st);
void launch_scale_to_f32(const void* src, int dtype, int64_t n, double scale, float* dst, cudaStream_t st);

// ---- multi-tensor optimizer step (adamw.cu): every owned slice of every parameter is cut
// into chunks of <= kOptChunk elements; one launch covers a list of chunk ids.
constexpr int64_t kOptChunk = 1 << 16;
struct OptSeg {
    const void* grad;  // synced owned grad slice (grad dtype)
    void* wout;        // owned slice of the weight (weight dtype)
    float* master;
    float* m;
    float* v;
    int64_t n;
    float scale;  // (float)(1/g), optim.cpp:155
    int vec;      // bf16 grad + bf16 weight, 16/8-byte aligned, n % 4 == 0: the x4 fast path
};
struct OptChunk {
    int64_t begin, len;
    int32_t seg, pad;
};
struct OptStepArgs {
    double lr, beta1, beta2, eps, weight_decay, bc1, bc2;
    double clip_norm;
    int clip_active, grad_dtype, weight_dtype, round_bf16;
};
// partials[ids[b]] = sum over chunk ids[b] of (float)(g*scale)^2 in fp64; non-finite grads
// set *nonfinite (the soft-failure scan of reliability.cpp:706-723, fused into this pass)
void launch_sumsq_chunks(const OptSeg* segs, const OptChunk* chunks, const int32_t* ids, int nids, int grad_dtype,
                         double* partials, int32_t* nonfinite, cudaStream_t st);
// *norm_sq = fixed-order sum of partials[0, n)
void launch_norm_final(const double* partials, int n, double* norm_sq, cudaStream_t st);
// fused unscale + clip (from *norm_sq) + AdamW + bf16 recast over the listed chunks. Like the
// reference's step (optim.cpp:130-194) it always applies the update; non-finite gradients are
// reported by the scan (StepStats.nonfinite / detect_soft_failure), which the training loop
// checks before stepping (train.cpp:193-194)
// sm_reserve > 0: the persistent grid leaves that many SMs free (for concurrent NCCL kernels)
void launch_adamw_chunks(const OptSeg* segs, const OptChunk* chunks, const int32_t* ids, int nids,
                         const OptStepArgs& a, const double* norm_sq, cudaStream_t st, int sm_reserve = 0);
// any non-finite element in the n-element buffer -> *flag = 1
void launch_nonfinite_scan(const void* g, int dtype, int64_t n, int32_t* flag, cudaStream_t st);

}  // namespace b2
