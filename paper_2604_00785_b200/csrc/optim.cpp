// EP-aware sharded optimizer step (src/optim.cpp:109-194) on B200.
//
//   1. gradient sync: EPSO reduce-scatters expert grads over the EP-orthogonal DP
//      group and non-expert grads over the fused DP x EP group (build_shard_plan,
//      optim.cpp:52-72); SO / DDP keep the reference's extra EP / DP all-reduces
//      (optim.cpp:142-146). NCCL over NVLink; a group of one member is a no-op and
//      the grad buffer itself is the synced slice.
//   2. global norm: fp64 sum of squares over counted slices (optim.cpp:74-86,
//      160-166), all-reduced over WORLD on the device.
//   3. fused unscale (1/g) + clip (derived on the device) + AdamW + bf16 recast.
//   4. all-gather of the updated slices in place (optim.cpp:185-190).
// Nothing waits on the host unless the caller asks for the step statistics.
#include "optim.h"

#include <cmath>
#include <cstring>

#include "comm.h"
#include "kernels.h"

namespace b2 {

void AdamWConfig::validate() const {
    check(beta1 > 0 && beta1 < 1 && beta2 > 0 && beta2 < 1, "adamw: betas must lie in (0,1)");
    check(eps > 0, "adamw: eps must be positive");
    check(min_lr <= peak_lr, "adamw: min_lr must not exceed peak_lr");
    check(warmup_steps >= 0 && total_steps >= warmup_steps, "adamw: need 0 <= warmup_steps <= total_steps");
}

double lr_at_step(int64_t step, const AdamWConfig& cfg) {
    check(step >= 0, "lr_at_step: negative step");
    if (step < cfg.warmup_steps) return cfg.peak_lr * (double)step / (double)cfg.warmup_steps;
    if (step >= cfg.total_steps) return cfg.min_lr;
    const double t = (double)(step - cfg.warmup_steps) / (double)(cfg.total_steps - cfg.warmup_steps);
    return cfg.min_lr + 0.5 * (cfg.peak_lr - cfg.min_lr) * (1.0 + std::cos(M_PI * t));
}

void shard_slice(int64_t numel, int group_size, int position, int64_t* begin, int64_t* end) {
    check(group_size >= 1 && position >= 0 && position < group_size, "shard_slice: bad position");
    const int64_t base = numel / group_size;
    *begin = (int64_t)position * base;
    *end = position == group_size - 1 ? numel : *begin + base;
}

static bool counts_toward_norm(ShardMode mode, bool expert, bool tp_sharded, const Context& c) {
    if (!tp_sharded && c.coord_tp != 0) return false;
    switch (mode) {
        case ShardMode::ddp: return c.coord_dp == 0 && (expert || c.coord_ep == 0);
        case ShardMode::so: return expert || c.coord_ep == 0;
        case ShardMode::epso: return true;
    }
    return false;
}

ShardedOptimizer::ShardedOptimizer(Context& ctx, const AdamWConfig& cfg, std::vector<ParamSlot> params,
                                   ShardMode mode, int weight_dtype, int grad_dtype)
    : ctx_(ctx), cfg_(cfg), params_(std::move(params)), mode_(mode), wdt_(weight_dtype), gdt_(grad_dtype) {
    cfg_.validate();
    check(wdt_ == F32 || wdt_ == BF16, "optimizer: weight dtype must be f32 or bf16");
    check(gdt_ == F32 || gdt_ == BF16, "optimizer: grad dtype must be f32 or bf16");
    check(ctx_.world == 1 || ctx_.comm != nullptr, "optimizer: multi-rank context without communicators");
    B2_CUDA(cudaSetDevice(ctx_.device));
    const size_t ge = dtype_size(gdt_);
    plan_.resize(params_.size());
    size_t bytes = 2 * 8 * (size_t)(nparts_ + 2) + 4096;
    for (size_t i = 0; i < params_.size(); ++i) {
        const ParamSlot& p = params_[i];
        check(p.weight && p.grad && p.numel >= 0, "shard plan: parameter needs matching weight/grad");
        Entry& e = plan_[i];
        if (mode_ == ShardMode::ddp) {
            e.own_b = 0;
            e.own_e = p.numel;
        } else {
            e.over_dp_ep = mode_ == ShardMode::epso && !p.expert;
            const int g = e.over_dp_ep ? ctx_.dp * ctx_.ep : ctx_.dp;
            const int pos = e.over_dp_ep ? ctx_.coord_dp * ctx_.ep + ctx_.coord_ep : ctx_.coord_dp;
            shard_slice(p.numel, g, pos, &e.own_b, &e.own_e);
        }
        e.counts = counts_toward_norm(mode_, p.expert, p.tp_sharded, ctx_);
        const int64_t n = e.own_e - e.own_b;
        bytes += 3 * (((size_t)n * 4 + 255) & ~size_t(255)) + 3 * 256;
        const bool pre_ep = !p.expert && mode_ != ShardMode::epso && ctx_.ep > 1;
        const int gsize = mode_ == ShardMode::ddp ? ctx_.dp : (e.over_dp_ep ? ctx_.dp * ctx_.ep : ctx_.dp);
        if (gsize > 1) bytes += (size_t)(mode_ == ShardMode::ddp ? p.numel : n) * ge + 512;
        if (pre_ep || mode_ == ShardMode::ddp) bytes += (size_t)p.numel * ge + 512;
    }
    arena_.reserve(bytes);
    norm_sq_ = arena_.take<double>(1);
    partials_ = arena_.take<double>(nparts_ + 1);
    for (size_t i = 0; i < params_.size(); ++i) {
        const ParamSlot& p = params_[i];
        Entry& e = plan_[i];
        const int64_t n = e.own_e - e.own_b;
        e.master = arena_.take<float>(n);
        e.m = arena_.take<float>(n);
        e.v = arena_.take<float>(n);
        // masters copied from the current weights, moments zero (optim.cpp:114-121)
        if (n > 0) {
            if (wdt_ == F32) {
                B2_CUDA(cudaMemcpyAsync(e.master, (const float*)p.weight + e.own_b, 4 * (size_t)n,
                                        cudaMemcpyDeviceToDevice, ctx_.stream));
            } else {
                launch_scale_to_f32((const __nv_bfloat16*)p.weight + e.own_b, BF16, n, 1.0, e.master, ctx_.stream);
            }
            B2_CUDA(cudaMemsetAsync(e.m, 0, 4 * (size_t)n, ctx_.stream));
            B2_CUDA(cudaMemsetAsync(e.v, 0, 4 * (size_t)n, ctx_.stream));
        }
        const bool pre_ep = !p.expert && mode_ != ShardMode::epso && ctx_.ep > 1;
        const int gsize = mode_ == ShardMode::ddp ? ctx_.dp : (e.over_dp_ep ? ctx_.dp * ctx_.ep : ctx_.dp);
        if (gsize > 1 && mode_ != ShardMode::ddp) e.scratch = arena_.take_bytes((size_t)n * ge);
        if (pre_ep || mode_ == ShardMode::ddp) e.scratch_full = arena_.take_bytes((size_t)p.numel * ge);
    }
    B2_CUDA(cudaStreamSynchronize(ctx_.stream));
}

ShardedOptimizer::~ShardedOptimizer() = default;

const Group* ShardedOptimizer::group_of(const Entry& e) const {
    if (!ctx_.comm) return nullptr;
    return e.over_dp_ep ? &ctx_.comm->dp_ep : &ctx_.comm->dp;
}

StepStats ShardedOptimizer::step(bool want_stats) {
    B2_CUDA(cudaSetDevice(ctx_.device));
    cudaStream_t st = ctx_.stream;
    launches_ = 0;
    StepStats stats;
    stats.step = step_count_;
    stats.lr = lr_at_step(step_count_, cfg_);
    const size_t ge = dtype_size(gdt_);
    // 1. gradient sync -> synced owned slice + its mean scale (optim.cpp:136-158)
    std::vector<const void*> synced(params_.size());
    std::vector<float> scale(params_.size(), 1.f);
    for (size_t i = 0; i < params_.size(); ++i) {
        const ParamSlot& p = params_[i];
        Entry& e = plan_[i];
        const void* src = p.grad;
        if (!p.expert && mode_ != ShardMode::epso && ctx_.ep > 1) {
            // allreduce_mean over EP (optim.cpp:142-143)
            all_reduce_sum(ctx_.comm->ep, p.grad, e.scratch_full, p.numel, nccl_dtype(gdt_), st);
            launch_scale_inplace(e.scratch_full, gdt_, p.numel, (float)(1.0 / (double)ctx_.ep), st);
            ++launches_;
            src = e.scratch_full;
        }
        if (mode_ == ShardMode::ddp) {
            if (ctx_.dp > 1) {
                all_reduce_sum(ctx_.comm->dp, src, e.scratch_full, p.numel, nccl_dtype(gdt_), st);
                src = e.scratch_full;
            }
            synced[i] = src;
            scale[i] = (float)(1.0 / (double)ctx_.dp);
        } else {
            const Group* g = group_of(e);
            const int gsize = e.over_dp_ep ? ctx_.dp * ctx_.ep : ctx_.dp;
            if (gsize > 1) {
                reduce_scatter_v(*g, src, e.scratch, p.numel, gdt_, st);
                synced[i] = e.scratch;
            } else {
                synced[i] = (const char*)src + (size_t)e.own_b * ge;
            }
            scale[i] = (float)(1.0 / (double)gsize);
        }
    }
    // 2. global grad norm over counted slices, all-reduced over WORLD (optim.cpp:160-166)
    bool first = true;
    for (size_t i = 0; i < params_.size(); ++i) {
        const Entry& e = plan_[i];
        if (!e.counts) continue;
        launch_sumsq_acc(synced[i], gdt_, e.own_e - e.own_b, scale[i], partials_, nparts_, norm_sq_, first, st);
        launches_ += 2;
        first = false;
    }
    if (first) B2_CUDA(cudaMemsetAsync(norm_sq_, 0, 8, st));
    if (ctx_.world > 1) all_reduce_sum(ctx_.comm->world, norm_sq_, norm_sq_, 1, ncclFloat64, st);
    const bool clip_active = !cfg_.clip_after_warmup_only || step_count_ >= cfg_.warmup_steps;
    // 3. fused unscale + clip + AdamW + bf16 recast on the owned slices (optim.cpp:174-184)
    const double bc1 = 1.0 - std::pow(cfg_.beta1, (double)(step_count_ + 1));
    const double bc2 = 1.0 - std::pow(cfg_.beta2, (double)(step_count_ + 1));
    for (size_t i = 0; i < params_.size(); ++i) {
        const ParamSlot& p = params_[i];
        Entry& e = plan_[i];
        AdamWKernelArgs a{};
        a.master = e.master;
        a.m = e.m;
        a.v = e.v;
        a.grad = synced[i];
        a.weight_out = (char*)p.weight + (size_t)e.own_b * dtype_size(wdt_);
        a.n = e.own_e - e.own_b;
        a.grad_dtype = gdt_;
        a.weight_dtype = wdt_;
        a.lr = stats.lr;
        a.beta1 = cfg_.beta1;
        a.beta2 = cfg_.beta2;
        a.eps = cfg_.eps;
        a.weight_decay = cfg_.weight_decay;
        a.bc1 = bc1;
        a.bc2 = bc2;
        a.grad_scale = scale[i];
        a.round_bf16 = cfg_.round_weights_bf16 ? 1 : 0;
        launch_adamw_full(a, norm_sq_, cfg_.clip_norm, clip_active ? 1 : 0, st);
        ++launches_;
        // 4. re-share (optim.cpp:185-190)
        if (mode_ != ShardMode::ddp) {
            const int gsize = e.over_dp_ep ? ctx_.dp * ctx_.ep : ctx_.dp;
            if (gsize > 1) all_gather_v(*group_of(e), p.weight, p.numel, wdt_, st);
        }
    }
    if (want_stats) {
        double sq = 0;
        B2_CUDA(cudaMemcpyAsync(&sq, norm_sq_, 8, cudaMemcpyDeviceToHost, st));
        B2_CUDA(cudaStreamSynchronize(st));
        stats.grad_norm = std::sqrt(sq);
        if (clip_active && stats.grad_norm > cfg_.clip_norm && stats.grad_norm > 0)
            stats.clip_scale = cfg_.clip_norm / stats.grad_norm;
    }
    step_count_++;
    return stats;
}

int64_t ShardedOptimizer::state_bytes() const {
    int64_t owned = 0;
    for (const Entry& e : plan_) owned += e.own_e - e.own_b;
    return 12 * owned;
}

void ShardedOptimizer::owned(int p, int64_t* b, int64_t* e) const {
    check(p >= 0 && p < (int)plan_.size(), "optimizer: parameter index out of range");
    *b = plan_[(size_t)p].own_b;
    *e = plan_[(size_t)p].own_e;
}

void ShardedOptimizer::get_state(int p, float* master, float* m, float* v) {
    check(p >= 0 && p < (int)plan_.size(), "optimizer: parameter index out of range");
    const Entry& e = plan_[(size_t)p];
    const size_t n = (size_t)(e.own_e - e.own_b);
    if (n == 0) return;
    if (master) B2_CUDA(cudaMemcpyAsync(master, e.master, 4 * n, cudaMemcpyDeviceToHost, ctx_.stream));
    if (m) B2_CUDA(cudaMemcpyAsync(m, e.m, 4 * n, cudaMemcpyDeviceToHost, ctx_.stream));
    if (v) B2_CUDA(cudaMemcpyAsync(v, e.v, 4 * n, cudaMemcpyDeviceToHost, ctx_.stream));
    B2_CUDA(cudaStreamSynchronize(ctx_.stream));
}

}  // namespace b2
