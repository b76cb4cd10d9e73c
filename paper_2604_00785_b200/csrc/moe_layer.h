// C++ host side of the B200 FastSparseMoE layer: the reference operator API
// (fast_moe_forward / fast_moe_backward / moe_aux_probs_grad / moe_aux_loss over a
// FastMoeState, include/optimus/moe.hpp:302-466) on device pointers.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <memory>
#include <vector>

#include "b2_common.cuh"

namespace b2 {

struct Sm100GemmArgs;

struct MoeConfig {  // moe.hpp:13-31
    int64_t n_experts = 8, top_k = 2, hidden = 64, intermediate = 128;
    int ep = 1;
    int64_t token_block = 8;
    bool normalize_topk = false;
    int64_t experts_per_rank() const { return n_experts / ep; }
    void validate() const;
};

struct Comm;  // ep collectives (comm.cpp); null for ep == 1

// One CUDA device + stream per rank (the reference's RankCtx, comm.hpp:205-231).
struct Context {
    int device = 0;
    cudaStream_t stream = nullptr;
    int num_sms = 148;
    int rank = 0, world = 1;
    int dp = 1, ep = 1, tp = 1, pp = 1;
    int coord_dp = 0, coord_ep = 0, coord_tp = 0, coord_pp = 0;
    Comm* comm = nullptr;
};

// Bump allocator over one device allocation (workspace lives as long as the layer), or
// over borrowed memory (adopt: a workspace shared by several layers).
class Arena {
  public:
    Arena() = default;
    ~Arena();
    Arena(const Arena&) = delete;
    Arena& operator=(const Arena&) = delete;
    void reserve(size_t bytes);
    void adopt(char* base, size_t cap);  // not owned: the caller keeps it alive
    template <typename T>
    T* take(int64_t n) {
        return static_cast<T*>(take_bytes((size_t)std::max<int64_t>(n, 1) * sizeof(T)));
    }
    void* take_bytes(size_t bytes);
    size_t used() const { return off_; }

  private:
    char* base_ = nullptr;
    size_t cap_ = 0, off_ = 0;
    bool owned_ = true;
};

// Device memory of the per-step activations of a layer; layers may share one (activation
// checkpointing: each backward replays its forward into the shared workspace).
struct Workspace {
    char* base = nullptr;
    size_t cap = 0;
    ~Workspace();
};

// FastMoeState (moe.hpp:302-316) plus the device workspace of one MoE layer on one rank.
class MoeLayer {
  public:
    // share_ws: reuse that layer's activation workspace (it must be large enough);
    // checkpoint: moe_block_forward's `ckpt` (blocks.cpp:339-377) — after forward only the
    // input pointer and the balancing statistics are held, and backward replays the forward
    // (its EP collectives included) before differentiating, bitwise like the reference.
    MoeLayer(Context& ctx, const MoeConfig& cfg, int dtype, int64_t max_tokens, const MoeLayer* share_ws = nullptr,
             bool checkpoint = false);
    ~MoeLayer();

    // fast_moe_forward (moe.hpp:344-390). All pointers are device pointers of `dtype`.
    void forward(const void* x, const void* router, const void* gate, const void* up, const void* down, int64_t s,
                 bool fur, void* out);
    // fast_moe_backward (moe.hpp:392-466). aux_probs_grad: [S, N] fp32 device or null.
    void backward(const void* router, const void* gate, const void* up, const void* down, const void* dout,
                  const float* aux_probs_grad, void* dx, void* drouter, void* dgate, void* dup, void* ddown);
    // moe_aux_probs_grad (moe.hpp:331-342) into a [S, N] fp32 device buffer
    void aux_probs_grad(double coeff, float* out);
    // moe_aux_loss (moe.hpp:320-328); synchronises the stream
    double aux_loss();

    // host copies of the state for parity checks (synchronise the stream)
    struct HostArtifacts {
        int64_t t_total = 0, th = 0, rt = 0, padded_rows = 0;
        std::vector<int64_t> token_counts, partial_token_counts, partial_cum, cum_token_counts, expert_counts,
            cum_expert_counts, input_indices, output_indices, selected_k, counter, pad_start;
    };
    HostArtifacts artifacts();
    void routing(float* probs, float* weights, int64_t* indices);  // local rows, host buffers
    void mean_probs_sel(float* mean_probs, int64_t* sel_counts);

    const MoeConfig& cfg() const { return cfg_; }
    int dtype() const { return dtype_; }
    int64_t pmax() const { return pmax_; }
    int64_t tokens() const { return s_; }
    size_t workspace_bytes() const { return ws_arena_.used() + arena_.used(); }
    // bytes this layer holds between forward and backward (the reference's MoeRec::held):
    // the persistent state, plus the workspace unless the layer checkpoints
    size_t held_bytes() const;
    bool checkpointing() const { return checkpoint_; }
    // number of kernels of this library launched by the last forward / backward
    int last_launches() const { return launches_; }

    // per-stage CUDA-event timing (profiling mode): 1 = eager launches, the mean over every
    // forward+backward since enabling; 2 = inside the CUDA graphs (event-record nodes around
    // each stage), the times of the last replayed forward+backward
    enum Stage {
        kRoute, kIndex, kGather, kGemmGateUp, kGemmDown, kCombine, kOutRedBwd, kGemmDgrad, kGemmWgradDown,
        kGemmWgradGateUp, kGemmDx, kRouterBwd, kNumStages
    };
    static const char* stage_name(int s);
    void set_profiling(int mode);
    void stage_times(float* ms);  // synchronises

    // CUDA-graph mode: a forward (backward) whose arguments repeat the previous call's is
    // captured once on the rank's stream and replayed as one graph launch afterwards.
    // Every data-dependent size lives on the device, so a replay is exact. Profiling
    // runs eagerly.
    void set_graph(bool on);
    void set_overlap_return(bool on) {
        overlap_opt_ = on;
        set_graph(graph_);
    }
  private:
    template <typename T>
    void forward_t(const T* x, const T* router, const T* gate, const T* up, const T* down, bool fur, T* out);
    template <typename T>
    void backward_t(const T* router, const T* gate, const T* up, const T* down, const T* dout,
                    const float* aux_probs_grad, T* dx, T* drouter, T* dgate, T* dup, T* ddown);

    void mark(int stage, bool end);
    void check_expert_ids();  // throws ContractError if an index kernel flagged an id outside [0, N)
    // partial weight-gradient dots per padded row left by the dgrad epilogue (one per 64 columns of I)
    int64_t wparts() const { return ceil_div(cfg_.intermediate, (int64_t)64); }
    void set_dispatch_tables();
    struct GraphCache {
        std::vector<const void*> key;
        int launches = 0;
        bool seen = false;
        cudaGraphExec_t exec = nullptr;
        void reset();
    };
    // eager the first time `key` is seen, captured the second time, replayed after that;
    // two entries per direction so double-buffered callers (the pipelined host-buffer
    // entry point alternates two staging slots) replay both
    static constexpr int kGraphSlots = 2;
    template <typename F>
    void run_graphed(GraphCache (&gcs)[kGraphSlots], std::vector<const void*> key, F&& body);
    bool graph_ = false;
    GraphCache gfwd_[kGraphSlots], gbwd_[kGraphSlots];
    int graph_lru_[2] = {0, 0};  // next slot to evict, per direction

    Context& ctx_;
    MoeConfig cfg_;
    int profiling_ = 0;
    int prof_step_ = -1;  // index of the profiled forward+backward being recorded
    std::vector<std::vector<cudaEvent_t>> prof_ev_;  // [step][stage*2 + end]
    int dtype_;
    int64_t smax_, tmax_, pmax_, thmax_;
    int64_t s_ = 0, t_ = 0, th_ = 0;
    bool fur_ = false, have_fwd_ = false;
    const void* x_ = nullptr;  // the caller's input, kept for the router weight-gradient
    int launches_ = 0;
    Arena arena_;     // persistent per-layer state (balancing statistics, flags)
    Arena ws_arena_;  // activations, routing artifacts, scratch: in ws_ (maybe shared)
    std::shared_ptr<Workspace> ws_;
    bool checkpoint_ = false;
    void* replay_out_ = nullptr;  // forward output of the checkpoint replay (discarded)
    // fp32
    float *logits_, *probs_, *topw_, *fw_, *colsum_, *mean_probs_, *wgrad_, *dlogits_, *dw_part_;
    // int32
    int32_t *topi_, *fi_, *sel_, *whist_, *wbase_, *expert_counts_, *cec_, *partial_counts_, *partial_cum_,
        *token_counts_, *ctc_, *pad_start_, *input_indices_, *output_indices_, *selected_k_, *slot_prow_,
        *prow_src_, *err_;
    float* prow_w_ = nullptr;  // bf16: padded row -> routing weight (0 pad), the weighted-H scheme
    float* wpart_ = nullptr;   // bf16: [pmax, wparts()] dgrad-epilogue partial dots
    int32_t* expert_order_ = nullptr;  // bf16: local experts by descending rows (wgrad tile order)
    const float* gw_ = nullptr;    // dispatch weights (learned or FUR)
    const int32_t* gi_ = nullptr;  // dispatch indices
    // dtype buffers (padded row space)
    void *mlp_in_, *g_, *u_, *h_, *y_, *dy_, *dh_, *dgu_, *dxp_;
    void* dl_bf16_ = nullptr;  // bf16 dlogits for the tensor-core router GEMMs
    void* dl_lo_ = nullptr;    // bf16(dlogits - dl_bf16_): low half of RouterDx's two-term split
    // expert parallelism (ep > 1) over NVLink peer memory: a symmetric CUDA-IPC buffer per
    // rank holds x / dout (pulled by the expert owners) and the return slabs the owners
    // store into; only the [S,K] routing table goes through an NCCL all-gather
    void ep_setup();
    void ep_barrier(cudaStream_t st = nullptr);
    // bf16, EP > 1: the backward returns dX / top-k weight gradients on a side stream while
    // the weight-gradient GEMMs run on num_sms - kCommSms SMs. Measured with the wide GEMM tiles
    // (tools/timeline.py --graph, same 4-GPU box): EP 4: 8 / 16 / 32 / 48 / 64 SMs 6.41 / 6.05 /
    // 5.66 / 5.77 / 5.98 ms per step, serial return 5.76; EP 2: serial 5.04-5.06 against 5.17-5.29
    // with 32 SMs — so the return overlaps from EP 4 up and runs after the GEMMs at EP 2
    bool overlap_return() const;
    // programmatic dependent launch inside the layer's graphs: on with EP (the NVLink kernels'
    // early launch pays: EP 4 5.62-5.65 vs 5.71 ms per step), off on one GPU, where the early-
    // resident dependents cost about what the hidden prologues save (17 alternated rounds on
    // four boxes: -60 us per step on average, single rounds from -240 to +70 us; in 100-step
    // runs held at the power cap (~1.45 GHz) the two are within 15 us)
    bool pdl_for_layer() const { return cfg_.ep > 1; }
    static constexpr int kCommSms = 32;
    static constexpr int kOverlapMinEp = 4;
    bool overlap_opt_ = true;
    cudaStream_t side_ = nullptr;
    cudaEvent_t ev_fork_ = nullptr, ev_join_ = nullptr;
    const int32_t* gi_local_ = nullptr;  // this rank's dispatch table [S,K] (learned or FUR)
    char* sym_ = nullptr;
    std::vector<char*> peer_base_;
    std::vector<char> peer_ipc_;  // 1: mapped through CUDA IPC (another process), 0: same process
    void** peer_tab_ = nullptr;  // device: tables of E pointers: x, dout, ret_f, ret_b, wret
    void *x_sh_ = nullptr, *dout_sh_ = nullptr, *ret_f_ = nullptr, *ret_b_ = nullptr;
    float* wret_ = nullptr;
    int* flags_ = nullptr;  // NVLink barrier counters (one per peer), in the symmetric buffer
    int32_t* tab_ids_ = nullptr;  // this rank's published routing table [S,K] (symmetric buffer)
    float* tab_w_ = nullptr;
    int32_t* gi_all_ = nullptr;
    float* gw_all_ = nullptr;
    int32_t* bar_ = nullptr;
    int32_t* colsum_ctr_ = nullptr;  // arrival counter of the fused mean_probs reduction (self-resetting)
    float* wgrad_local_ = nullptr;
    void* dx_exp_ = nullptr;
};

}  // namespace b2
