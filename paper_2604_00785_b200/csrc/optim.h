// EP-aware sharded AdamW on B200: ShardedOptimizer (include/optimus/optim.hpp:98-121,
// src/optim.cpp:109-194) over device-resident weights/grads with NCCL collectives.
#pragma once
#include <stdint.h>

#include <vector>

#include "comm.h"
#include "kernels.h"
#include "moe_layer.h"

namespace b2 {

struct AdamWConfig {  // optim.hpp:11-25
    double beta1 = 0.9, beta2 = 0.99, eps = 1e-8, weight_decay = 0.1, peak_lr = 4e-4, min_lr = 4e-5;
    int64_t warmup_steps = 2500, total_steps = 100000;
    double clip_norm = 1.0;
    bool clip_after_warmup_only = true, round_weights_bf16 = true;
    void validate() const;
};

double lr_at_step(int64_t step, const AdamWConfig& cfg);
void shard_slice(int64_t numel, int group_size, int position, int64_t* begin, int64_t* end);
// memory_report (optim.cpp:196-221): the 16P-per-parameter footprint (bf16 weights and grads,
// fp32 master + two moments divided over the owning group) against a device capacity
struct MemoryReport {
    double weights_bytes = 0, grads_bytes = 0, master_bytes = 0, optim_bytes = 0;
    double total_bytes = 0, capacity_bytes = 0;
    bool feasible = true;
};
MemoryReport memory_report(int64_t p_expert, int64_t p_non_expert, int mode, int dp, int ep, double capacity_gb);

enum class ShardMode { ddp = 0, so = 1, epso = 2 };

struct ParamSlot {
    void* weight = nullptr;
    const void* grad = nullptr;
    int64_t numel = 0;
    bool expert = false;
    bool tp_sharded = false;
};

struct StepStats {
    int64_t step = 0;
    double lr = 0, grad_norm = 0, clip_scale = 1.0;
    int nonfinite = 0;  // a grad held NaN/Inf (the fused scan); the update was applied, as the reference's
};

class ShardedOptimizer {
  public:
    ShardedOptimizer(Context& ctx, const AdamWConfig& cfg, std::vector<ParamSlot> params, ShardMode mode,
                     int weight_dtype, int grad_dtype);
    ~ShardedOptimizer();
    // want_stats: copy the norm back (synchronises); otherwise fully asynchronous
    StepStats step(bool want_stats);
    int64_t state_bytes() const;
    void owned(int p, int64_t* b, int64_t* e) const;
    void get_state(int p, float* master, float* m, float* v);
    // checkpoint assembly (reliability.cpp:411-440): the FULL master / exp_avg / exp_avg_sq of
    // param p, gathered over its owning group (collective on that group; host buffers of numel)
    void gather_state(int p, float* master, float* m, float* v);
    // restore (reliability.cpp:658-667): this rank's owned slice from full host tensors
    void load_state(int p, const float* master, const float* m, const float* v);
    // device variants for the record-file checkpoint (ckpt_state.cpp): full fp32 tensors
    // gathered into device buffers of numel floats (NULL skips one) / the owned slices
    void gather_state_device(int p, float* master, float* m, float* v);
    void state_slices(int p, float** master, float** m, float** v) const;
    int num_params() const { return (int)params_.size(); }
    const ParamSlot& param(int p) const { return params_[(size_t)p]; }
    bool over_dp_ep(int p) const { return plan_[(size_t)p].over_dp_ep; }
    int weight_dtype() const { return wdt_; }
    int grad_dtype() const { return gdt_; }
    Context& context() { return ctx_; }
    int64_t step_count() const { return step_count_; }
    void set_step_count(int64_t n) { step_count_ = n; }
    int last_launches() const { return launches_; }
    // detect_soft_failure (reliability.cpp:706-723): scans this rank's LOCAL grads (and
    // the loss) for NaN/Inf and max-all-reduces (node + 1) over WORLD; returns the
    // highest sick node or -1. Synchronises.
    int detect_soft_failure(double loss, int node);

  private:
    struct Entry {
        int64_t own_b = 0, own_e = 0;
        bool over_dp_ep = false;
        bool counts = true;
        float *master = nullptr, *m = nullptr, *v = nullptr;
        void* scratch = nullptr;       // synced owned slice (grad dtype), when the group has > 1 member
        void* scratch_full = nullptr;  // SO/DDP pre-reduction buffer
    };
    const Group* group_of(const Entry& e) const;
    Context& ctx_;
    AdamWConfig cfg_;
    std::vector<ParamSlot> params_;
    ShardMode mode_;
    int wdt_, gdt_;
    std::vector<Entry> plan_;
    Arena arena_;
    double* norm_sq_ = nullptr;  // device
    double* partials_ = nullptr;  // one fp64 partial per chunk, param-major (fixed reduction order)
    int32_t* nonfinite_ = nullptr;
    int32_t* sick_ = nullptr;
    // multi-tensor tables: segments (one per param), chunks, and chunk-id lists per phase
    OptSeg* segs_ = nullptr;
    OptChunk* chunks_ = nullptr;
    int32_t *ids_local_norm_ = nullptr, *ids_pre_norm_ = nullptr, *ids_local_ = nullptr, *ids_pre_ = nullptr;
    int n_chunks_ = 0, n_local_norm_ = 0, n_pre_norm_ = 0, n_local_ = 0, n_pre_ = 0;
    std::vector<char> pre_;  // param needs a collective before its update
    cudaStream_t comm_stream_ = nullptr;
    cudaEvent_t ev_start_ = nullptr, ev_synced_ = nullptr, ev_pre_done_ = nullptr, ev_ag_ = nullptr;
    cudaEvent_t ev_pre_updated_ = nullptr;  // the synced parameters' update is done: re-share
    int64_t step_count_ = 0;
    int launches_ = 0;
};

}  // namespace b2
