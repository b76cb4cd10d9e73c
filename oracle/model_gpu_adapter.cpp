// TEST INFRASTRUCTURE ONLY — the model-level integration check of SURVEY §8(f)3.
//
// Linked into oracle/_ref/model_parity_gpu with -Wl,--wrap on the reference's two MoE block
// entry points, so the UNMODIFIED reference model (src/model.cpp chunk_forward /
// chunk_backward, src/blocks.cpp, the pipeline schedule, attention, norms, CE loss) runs with
// every MoE layer on the B200 through the C-ABI (include/b2moe.h) instead of
// fast_moe_forward / fast_moe_backward:
//   moe_block_forward   blocks.cpp:339-355  -> b2_moe_forward + b2_moe_aux_loss + artifacts
//   moe_block_backward  blocks.cpp:357-377  -> b2_moe_aux_probs_grad + b2_moe_backward
//   ShardedOptimizer::step  optim.cpp:130-194 -> b2_opt_step (when the driver registers the
//                           model's slots with b2_adapter_use_gpu_optimizer: grads up, the fused
//                           EPSO AdamW on the device, bf16-rounded weights back)
// This is exactly the adapter INTEGRATION.md describes for a maintainer (fp32 layer — or the
// bf16 tensor-core layer with B2_ADAPTER_BF16=1 — one GPU state per MoeRec = per (layer,
// microbatch), host Tensor in / Tensor out; at EP > 1 each rank thread of the reference's World
// drives the GPU of its EP coordinate).
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "optimus/blocks.hpp"
#include "optimus/kernels.hpp"
#include "optimus/optim.hpp"
#include "../include/b2moe.h"

using namespace optimus;

namespace {

void ok(int rc, const char* what) {
    if (rc != B2_OK) throw std::runtime_error(std::string("b2 adapter: ") + what + ": " + b2_last_error());
}
void cu(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string("b2 adapter: ") + what + ": " + cudaGetErrorString(e));
}

// B2_ADAPTER_BF16=1: the bf16 layer (tcgen05 tensor-core GEMMs) instead of the fp32 one; the
// adapter rounds the fp32 tensors to bf16 (RNE) at the boundary and widens the results
bool bf16_mode() {
    static const bool on = [] {
        const char* e = std::getenv("B2_ADAPTER_BF16");
        return e && std::atoi(e) == 1;
    }();
    return on;
}
uint16_t to_bf16(float f) {
    uint32_t u;
    std::memcpy(&u, &f, 4);
    if ((u & 0x7fffffffu) > 0x7f800000u) return (uint16_t)((u >> 16) | 0x40u);
    return (uint16_t)((u + 0x7fffu + ((u >> 16) & 1u)) >> 16);
}

struct Dev {
    void* p = nullptr;
    int64_t n = 0;
    size_t es() const { return bf16_mode() ? 2 : 4; }
    void need(int64_t k) {
        if (k <= n) return;
        if (p) cudaFree(p);
        cu(cudaMalloc(&p, es() * (size_t)std::max<int64_t>(k, 1)), "cudaMalloc");
        n = k;
    }
    void up(const TensorF& t) {
        need(t.numel());
        if (!bf16_mode()) {
            cu(cudaMemcpy(p, t.data(), 4 * (size_t)t.numel(), cudaMemcpyHostToDevice), "H2D");
            return;
        }
        std::vector<uint16_t> h((size_t)t.numel());
        for (int64_t i = 0; i < t.numel(); ++i) h[(size_t)i] = to_bf16(t.data()[i]);
        cu(cudaMemcpy(p, h.data(), 2 * h.size(), cudaMemcpyHostToDevice), "H2D");
    }
    void down(TensorF& t) const {
        if (!bf16_mode()) {
            cu(cudaMemcpy(t.data(), p, 4 * (size_t)t.numel(), cudaMemcpyDeviceToHost), "D2H");
            return;
        }
        std::vector<uint16_t> h((size_t)t.numel());
        cu(cudaMemcpy(h.data(), p, 2 * h.size(), cudaMemcpyDeviceToHost), "D2H");
        for (int64_t i = 0; i < t.numel(); ++i) {
            const uint32_t u = (uint32_t)h[(size_t)i] << 16;
            std::memcpy(&t.data()[i], &u, 4);
        }
    }
};

struct GpuLayer {
    b2_moe* m = nullptr;
    int64_t cap = 0;
    Dev x, router, gate, up, down, out, dy, dx, dr, dg, du, dd;
    float* apg = nullptr;  // [S, N] fp32 in both modes
    int64_t apg_n = 0;
};

// EP > 1: the reference's rank threads each drive their own GPU (device = EP coordinate); the
// layer's EP exchange then runs over direct peer access between the threads' devices, its
// NCCL communicators from one id shared through this process
thread_local b2_ctx* g_ctx = nullptr;
thread_local std::map<const MoeRec*, GpuLayer> g_layers;  // one GPU state per (layer, microbatch)
std::once_flag g_id_once;
uint8_t g_nccl_id[128];

void ensure_ctx(const RankCtx& rc, int E) {
    if (g_ctx) return;
    if (E <= 1) {
        ok(b2_ctx_create(0, nullptr, 0, 1, 1, 1, 1, nullptr, &g_ctx), "ctx");
        return;
    }
    std::call_once(g_id_once, [] { ok(b2_nccl_unique_id(g_nccl_id), "nccl id"); });
    const int ep = rc.coord().ep;
    ok(b2_ctx_create(ep, nullptr, ep, 1, E, 1, 1, g_nccl_id, &g_ctx), "ctx (EP)");
}

GpuLayer& layer_for(const MoeRec* rec, const MoeConfig& cfg, int64_t S) {
    GpuLayer& L = g_layers[rec];
    if (!L.m || L.cap < S) {
        if (L.m) b2_moe_destroy(L.m);
        b2_moe_cfg c{cfg.n_experts, cfg.top_k, cfg.hidden, cfg.intermediate, (int32_t)cfg.ep,
                     cfg.normalize_topk ? 1 : 0, cfg.token_block};
        ok(b2_moe_create(g_ctx, &c, bf16_mode() ? B2_BF16 : B2_F32, S, &L.m), "create");
        L.cap = S;
    }
    return L;
}

void upload_weights(GpuLayer& L, const ExpertWeights<float>& w) {
    L.router.up(w.router);
    L.gate.up(w.gate);
    L.up.up(w.up);
    L.down.up(w.down);
}

}  // namespace

extern "C" {

// moe_block_forward (blocks.cpp:339-355) on the B200
TensorF __wrap__ZN7optimus17moe_block_forwardERNS_7RankCtxERKNS_12ProcessGroupERKNS_6TensorIfEERKNS_13ExpertWeightsIfEERKNS_9MoeConfigEbbRNS_6MoeRecEPNS_9ActLedgerEPNS_11ExpertTallyE(
    RankCtx& rctx, const ProcessGroup& ep_group, const TensorF& x, const ExpertWeights<float>& w, const MoeConfig& cfg,
    bool fur, bool ckpt, MoeRec& rec, ActLedger* led, ExpertTally* tally) {
    check(ep_group.size() == cfg.ep, "b2 adapter: cfg.ep must match the EP group");
    ensure_ctx(rctx, ep_group.size());
    const int64_t S = x.dim(0), H = cfg.hidden;
    GpuLayer& L = layer_for(&rec, cfg, S);
    rec.ckpt = ckpt;
    upload_weights(L, w);
    L.x.up(x);
    L.out.need(S * H);
    ok(b2_moe_forward(L.m, L.x.p, L.router.p, L.gate.p, L.up.p, L.down.p, S, fur ? 1 : 0, L.out.p), "forward");
    TensorF out({S, H});
    L.out.down(out);
    ok(b2_moe_aux_loss(L.m, &rec.aux), "aux loss");
    if (tally) {  // routed tokens per local expert (RoutingArtifacts::token_counts)
        const int64_t nr = cfg.n_experts / cfg.ep, T = S * cfg.ep, K = cfg.top_k;
        const int64_t th = (T + cfg.token_block - 1) / cfg.token_block;
        int64_t sizes[4];
        std::vector<int64_t> tc((size_t)nr), ptc((size_t)(nr * th + 1)), pc((size_t)(nr * th + 1)),
            ctc((size_t)nr + 1), ec((size_t)T), cec((size_t)T + 1), ii((size_t)(T * K)), oi((size_t)(T * K)),
            sk((size_t)(T * K)), cnt((size_t)(nr * th + 1));
        ok(b2_moe_artifacts(L.m, sizes, tc.data(), ptc.data(), pc.data(), ctc.data(), ec.data(), cec.data(), ii.data(),
                            oi.data(), sk.data(), cnt.data()),
           "artifacts");
        TensorI t({nr});
        std::memcpy(t.data(), tc.data(), sizeof(int64_t) * (size_t)nr);
        tally->accumulate(t);
    }
    rec.held = b2_moe_held_bytes(L.m);
    detail::led_charge(led, rec.held);
    return out;
}

// moe_block_backward (blocks.cpp:357-377) on the B200; grads accumulate into g like the reference
TensorF __wrap__ZN7optimus18moe_block_backwardERNS_7RankCtxERKNS_12ProcessGroupERKNS_13ExpertWeightsIfEERKNS_9MoeConfigEbdRNS_6MoeRecERKNS_6TensorIfEERNS_13MoeParamGradsEPNS_9ActLedgerE(
    RankCtx& rctx, const ProcessGroup& ep_group, const ExpertWeights<float>& w, const MoeConfig& cfg, bool,
    double aux_coeff, MoeRec& rec, const TensorF& dy, MoeParamGrads& g, ActLedger* led) {
    check(ep_group.size() == cfg.ep, "b2 adapter: cfg.ep must match the EP group");
    ensure_ctx(rctx, ep_group.size());
    const int64_t S = dy.dim(0), H = cfg.hidden;
    GpuLayer& L = layer_for(&rec, cfg, S);
    upload_weights(L, w);
    if (L.apg_n < S * cfg.n_experts) {
        if (L.apg) cudaFree(L.apg);
        cu(cudaMalloc((void**)&L.apg, 4 * (size_t)(S * cfg.n_experts)), "cudaMalloc");
        L.apg_n = S * cfg.n_experts;
    }
    ok(b2_moe_aux_probs_grad(L.m, aux_coeff, L.apg), "aux probs grad");
    L.dy.up(dy);
    L.dx.need(S * H);
    L.dr.need(w.router.numel());
    L.dg.need(w.gate.numel());
    L.du.need(w.up.numel());
    L.dd.need(w.down.numel());
    ok(b2_moe_backward(L.m, L.router.p, L.gate.p, L.up.p, L.down.p, L.dy.p, L.apg, L.dx.p, L.dr.p, L.dg.p, L.du.p,
                       L.dd.p),
       "backward");
    TensorF dx({S, H}), dr(w.router.shape()), dg(w.gate.shape()), du(w.up.shape()), dd(w.down.shape());
    L.dx.down(dx);
    L.dr.down(dr);
    L.dg.down(dg);
    L.du.down(du);
    L.dd.down(dd);
    add_inplace(g.router, dr);
    add_inplace(g.gate, dg);
    add_inplace(g.up, du);
    add_inplace(g.down, dd);
    detail::led_release(led, rec.held);
    rec = MoeRec{};
    return dx;
}

}  // extern "C"

// ---- the optimizer step on the B200 (optional: registered by the driver) ---------------------
namespace {
struct GpuOpt {
    b2_opt* o = nullptr;
    std::vector<ParamSlot> slots;
    std::vector<float*> w, g;
};
GpuOpt* g_opt = nullptr;
}  // namespace

// the driver hands over the model's slots and the AdamW config; masters come from the current
// weights, moments start at zero (optim.cpp:109-122)
void b2_adapter_use_gpu_optimizer(const std::vector<ParamSlot>& slots, const AdamWConfig& c) {
    if (!g_ctx) ok(b2_ctx_create(0, nullptr, 0, 1, 1, 1, 1, nullptr, &g_ctx), "ctx");  // EP = 1 only
    g_opt = new GpuOpt;
    g_opt->slots = slots;
    std::vector<b2_param> ps;
    for (const ParamSlot& s : slots) {
        float *w = nullptr, *g = nullptr;
        const int64_t n = s.weight->numel();
        cu(cudaMalloc((void**)&w, 4 * (size_t)n), "cudaMalloc");
        cu(cudaMalloc((void**)&g, 4 * (size_t)n), "cudaMalloc");
        cu(cudaMemcpy(w, s.weight->data(), 4 * (size_t)n, cudaMemcpyHostToDevice), "H2D");
        g_opt->w.push_back(w);
        g_opt->g.push_back(g);
        ps.push_back(b2_param{w, g, n, s.cls == ReplicationClass::expert ? 1 : 0, s.tp_sharded ? 1 : 0});
    }
    b2_adamw_cfg ac{c.beta1, c.beta2, c.eps, c.weight_decay, c.peak_lr, c.min_lr, c.warmup_steps, c.total_steps,
                    c.clip_norm, c.clip_after_warmup_only ? 1 : 0, c.round_weights_bf16 ? 1 : 0};
    ok(b2_opt_create(g_ctx, &ac, ps.data(), (int)ps.size(), B2_EPSO, B2_F32, B2_F32, &g_opt->o), "opt create");
}

extern "C" {
StepStats __real__ZN7optimus16ShardedOptimizer4stepEv(ShardedOptimizer* self);

// ShardedOptimizer::step (optim.cpp:130-194); the reference's own step when no GPU optimizer
// was registered
StepStats __wrap__ZN7optimus16ShardedOptimizer4stepEv(ShardedOptimizer* self) {
    if (!g_opt) return __real__ZN7optimus16ShardedOptimizer4stepEv(self);
    for (size_t i = 0; i < g_opt->slots.size(); ++i) {
        const TensorF& gr = *g_opt->slots[i].grad;
        cu(cudaMemcpy(g_opt->g[i], gr.data(), 4 * (size_t)gr.numel(), cudaMemcpyHostToDevice), "H2D");
    }
    b2_step_stats st{};
    ok(b2_opt_step(g_opt->o, &st), "opt step");
    for (size_t i = 0; i < g_opt->slots.size(); ++i) {
        TensorF& w = *g_opt->slots[i].weight;
        cu(cudaMemcpy(w.data(), g_opt->w[i], 4 * (size_t)w.numel(), cudaMemcpyDeviceToHost), "D2H");
    }
    StepStats out;
    out.step = st.step;
    out.lr = st.lr;
    out.grad_norm = st.grad_norm;
    out.clip_scale = st.clip_scale;
    return out;
}
}  // extern "C"
