// extern "C" entry points of include/b2moe.h over the C++ host classes.
#include "../../include/b2moe.h"

#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>

#include "ckpt_state.h"
#include "comm.h"
#include "kernels.h"
#include "moe_layer.h"
#include "optim.h"

using namespace b2;

namespace {
thread_local std::string g_last_error;

template <class F>
int guard(F&& f) {
    try {
        f();
        return B2_OK;
    } catch (const Error& e) {
        g_last_error = e.what();
        return e.code;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return B2_ERR_CONTRACT;
    }
}

MoeConfig to_cfg(const b2_moe_cfg* c) {
    check(c != nullptr, "moe: null config");
    MoeConfig m;
    m.n_experts = c->n_experts;
    m.top_k = c->top_k;
    m.hidden = c->hidden;
    m.intermediate = c->intermediate;
    m.ep = c->ep;
    m.token_block = c->token_block;
    m.normalize_topk = c->normalize_topk != 0;
    return m;
}

AdamWConfig to_acfg(const b2_adamw_cfg* a) {
    check(a != nullptr, "adamw: null config");
    AdamWConfig c;
    c.beta1 = a->beta1;
    c.beta2 = a->beta2;
    c.eps = a->eps;
    c.weight_decay = a->weight_decay;
    c.peak_lr = a->peak_lr;
    c.min_lr = a->min_lr;
    c.warmup_steps = a->warmup_steps;
    c.total_steps = a->total_steps;
    c.clip_norm = a->clip_norm;
    c.clip_after_warmup_only = a->clip_after_warmup_only != 0;
    c.round_weights_bf16 = a->round_weights_bf16 != 0;
    return c;
}

void require_device() {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) throw CudaError("no CUDA device: the B200 path has no CPU fallback");
}
}  // namespace

struct b2_ctx {
    Context c;
    std::unique_ptr<Comm> comm;
    bool own_stream = false;
    cudaStream_t copy_stream = nullptr;
};
// host-buffer entry point: two staging slots {x, dout, out, dx, aux grad} so step i+1's
// host->device copies run while step i computes and step i's results stream back
struct HostIo {
    char* dev = nullptr;
    size_t slot_bytes = 0;
    int64_t cap_tokens = -1;
    cudaStream_t h2d = nullptr, d2h = nullptr;
    cudaEvent_t ev_x[2] = {}, ev_in[2] = {}, ev_fwd[2] = {}, ev_bwd[2] = {}, ev_out[2] = {};
    bool used[2] = {false, false};
    int next = 0;
    bool warned_pageable = false;
};

// true when `p` is page-locked host memory (or device memory): its async copies do not block
static bool async_copy_ok(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost || a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}
struct b2_moe {
    b2_ctx* ctx;
    std::unique_ptr<MoeLayer> layer;
    HostIo io;
};
struct b2_opt {
    b2_ctx* ctx;
    std::unique_ptr<ShardedOptimizer> opt;
};

namespace b2 {
// programmatic dependent launch, on by default (the optimizer); MoeLayer turns it off for its
// single-GPU calls (b2_common.cuh PdlScope)
static thread_local bool g_pdl = true;
bool pdl_enabled() { return g_pdl; }
void set_pdl_enabled(bool on) { g_pdl = on; }
}  // namespace b2

extern "C" {

const char* b2_last_error(void) { return g_last_error.c_str(); }
const char* b2_version(void) { return "b2moe 0.1 (sm_100a tcgen05 grouped GEMM, fused EPSO AdamW)"; }

int b2_device_ok(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) return 0;
    return sm100_available() ? 1 : 0;
}

int b2_nccl_unique_id(uint8_t out[128]) {
    return guard([&] {
        ncclUniqueId id;
        B2_NCCL(ncclGetUniqueId(&id));
        std::memcpy(out, &id, 128);
    });
}

int b2_ctx_create(int device, void* stream, int rank, int dp, int ep, int tp, int pp, const uint8_t* nccl_id,
                  b2_ctx** out) {
    return guard([&] {
        require_device();
        check(dp >= 1 && ep >= 1 && tp >= 1 && pp >= 1, "topology: axes must be >= 1");
        const int world = dp * ep * tp * pp;
        check(rank >= 0 && rank < world, "ctx: rank out of range");
        auto c = std::make_unique<b2_ctx>();
        Context& x = c->c;
        x.device = device;
        B2_CUDA(cudaSetDevice(device));
        // the caller's stream; NULL is the legacy default stream, so work stays ordered
        // with a framework (e.g. torch) that launches on it
        x.stream = (cudaStream_t)stream;
        B2_CUDA(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
        B2_CUDA(cudaDeviceGetAttribute(&x.num_sms, cudaDevAttrMultiProcessorCount, device));
        x.rank = rank;
        x.world = world;
        x.dp = dp;
        x.ep = ep;
        x.tp = tp;
        x.pp = pp;
        int r = rank;  // coord_of (comm.hpp:49-59)
        x.coord_tp = r % tp;
        r /= tp;
        x.coord_ep = r % ep;
        r /= ep;
        x.coord_dp = r % dp;
        r /= dp;
        x.coord_pp = r;
        if (world > 1) {
            check(nccl_id != nullptr, "ctx: world > 1 needs an NCCL unique id");
            c->comm.reset(comm_create(nccl_id, rank, dp, ep, tp, pp, x.coord_dp, x.coord_ep, x.coord_tp, x.coord_pp,
                                      device));
            x.comm = c->comm.get();
        }
        *out = c.release();
    });
}

int b2_ctx_destroy(b2_ctx* ctx) {
    return guard([&] {
        if (!ctx) return;
        cudaStreamSynchronize(ctx->c.stream);
        ctx->comm.reset();
        if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
        if (ctx->own_stream) cudaStreamDestroy(ctx->c.stream);
        delete ctx;
    });
}

int b2_ctx_sync(b2_ctx* ctx) { return guard([&] { B2_CUDA(cudaStreamSynchronize(ctx->c.stream)); }); }

int b2_moe_create_ex(b2_ctx* ctx, const b2_moe_cfg* cfg, int dtype, int64_t max_tokens, const b2_moe* share_workspace,
                     int checkpoint, b2_moe** out) {
    return guard([&] {
        check(ctx != nullptr, "moe: null context");
        auto m = std::make_unique<b2_moe>();
        m->ctx = ctx;
        if (dtype == BF16) check(sm100_available(), "bf16 expert path needs an sm_100 (B200) device");
        m->layer = std::make_unique<MoeLayer>(ctx->c, to_cfg(cfg), dtype, max_tokens,
                                              share_workspace ? share_workspace->layer.get() : nullptr,
                                              checkpoint != 0);
        *out = m.release();
    });
}

int b2_moe_create(b2_ctx* ctx, const b2_moe_cfg* cfg, int dtype, int64_t max_tokens, b2_moe** out) {
    return b2_moe_create_ex(ctx, cfg, dtype, max_tokens, nullptr, 0, out);
}

int64_t b2_moe_held_bytes(b2_moe* m) { return m ? (int64_t)m->layer->held_bytes() : -1; }

int b2_moe_destroy(b2_moe* m) {
    return guard([&] {
        if (!m) return;
        cudaStreamSynchronize(m->ctx->c.stream);
        HostIo& io = m->io;
        if (io.h2d) cudaStreamSynchronize(io.h2d);
        if (io.d2h) cudaStreamSynchronize(io.d2h);
        if (io.dev) cudaFree(io.dev);
        for (int b = 0; b < 2; ++b)
            for (cudaEvent_t e : {io.ev_x[b], io.ev_in[b], io.ev_fwd[b], io.ev_bwd[b], io.ev_out[b]})
                if (e) cudaEventDestroy(e);
        if (io.h2d) cudaStreamDestroy(io.h2d);
        if (io.d2h) cudaStreamDestroy(io.d2h);
        delete m;
    });
}

int b2_moe_forward(b2_moe* m, const void* x, const void* router, const void* gate, const void* up, const void* down,
                   int64_t s_tokens, int fur, void* out) {
    return guard([&] { m->layer->forward(x, router, gate, up, down, s_tokens, fur != 0, out); });
}

int b2_moe_backward(b2_moe* m, const void* router, const void* gate, const void* up, const void* down,
                    const void* dout, const float* aux_probs_grad, void* dx, void* drouter, void* dgate, void* dup,
                    void* ddown) {
    return guard([&] { m->layer->backward(router, gate, up, down, dout, aux_probs_grad, dx, drouter, dgate, dup, ddown); });
}

int b2_moe_aux_probs_grad(b2_moe* m, double coeff, float* out) {
    return guard([&] { m->layer->aux_probs_grad(coeff, out); });
}

int b2_moe_aux_loss(b2_moe* m, double* out) { return guard([&] { *out = m->layer->aux_loss(); }); }

int b2_moe_routing(b2_moe* m, float* probs_host, float* weights_host, int64_t* indices_host) {
    return guard([&] { m->layer->routing(probs_host, weights_host, indices_host); });
}

static void copy_artifacts(const MoeLayer::HostArtifacts& a, int64_t* sizes, int64_t* token_counts,
                           int64_t* partial_token_counts, int64_t* partial_cum, int64_t* cum_token_counts,
                           int64_t* expert_counts, int64_t* cum_expert_counts, int64_t* input_indices,
                           int64_t* output_indices, int64_t* selected_k, int64_t* counter) {
    sizes[0] = a.t_total;
    sizes[1] = a.th;
    sizes[2] = a.rt;
    sizes[3] = a.padded_rows;
    auto cp = [](int64_t* dst, const std::vector<int64_t>& v) {
        if (dst && !v.empty()) std::memcpy(dst, v.data(), 8 * v.size());
    };
    cp(token_counts, a.token_counts);
    cp(partial_token_counts, a.partial_token_counts);
    cp(partial_cum, a.partial_cum);
    cp(cum_token_counts, a.cum_token_counts);
    cp(expert_counts, a.expert_counts);
    cp(cum_expert_counts, a.cum_expert_counts);
    cp(input_indices, a.input_indices);
    cp(output_indices, a.output_indices);
    cp(selected_k, a.selected_k);
    cp(counter, a.counter);
}

int b2_moe_artifacts(b2_moe* m, int64_t* sizes_host, int64_t* token_counts, int64_t* partial_token_counts,
                     int64_t* partial_cum, int64_t* cum_token_counts, int64_t* expert_counts,
                     int64_t* cum_expert_counts, int64_t* input_indices, int64_t* output_indices,
                     int64_t* selected_k, int64_t* counter) {
    return guard([&] {
        copy_artifacts(m->layer->artifacts(), sizes_host, token_counts, partial_token_counts, partial_cum,
                       cum_token_counts, expert_counts, cum_expert_counts, input_indices, output_indices, selected_k,
                       counter);
    });
}

// Enqueues one forward+backward over host buffers on a two-slot pipeline:
//   h2d stream : [wait: slot's previous backward] x (ev_x), dout -> slot (ev_in)
//   compute    : [wait ev_x, slot's previous out/dx read-back] forward (ev_fwd), [wait ev_in]
//                aux grad, backward (ev_bwd)
//   d2h stream : [wait ev_fwd] out -> host, [wait ev_bwd] dx -> host       (ev_out)
static void fwd_bwd_host_enqueue(b2_moe* m, const void* x_host, const void* dout_host, const void* router,
                                 const void* gate, const void* up, const void* down, double aux_coeff,
                                 void* out_host, void* dx_host, void* drouter, void* dgate, void* dup, void* ddown,
                                 int64_t s_tokens) {
    MoeLayer& L = *m->layer;
    const MoeConfig& c = L.cfg();
    Context& cx = m->ctx->c;
    HostIo& io = m->io;
    B2_CUDA(cudaSetDevice(cx.device));
    const size_t es = dtype_size(L.dtype());
    const size_t tok_bytes = (size_t)s_tokens * (size_t)c.hidden * es;
    const size_t aux_bytes = sizeof(float) * (size_t)std::max<int64_t>(1, c.n_experts * s_tokens);
    if (io.cap_tokens < s_tokens) {  // (re)size the staging slots: drain the pipeline first
        for (cudaStream_t q : {cx.stream, io.h2d, io.d2h})
            if (q) B2_CUDA(cudaStreamSynchronize(q));
        if (io.dev) B2_CUDA(cudaFree(io.dev));
        io.slot_bytes = ((4 * tok_bytes + aux_bytes + 255) & ~size_t(255));
        B2_CUDA(cudaMalloc((void**)&io.dev, 2 * std::max<size_t>(io.slot_bytes, 256)));
        io.cap_tokens = s_tokens;
        io.used[0] = io.used[1] = false;
        if (!io.h2d) {
            B2_CUDA(cudaStreamCreateWithFlags(&io.h2d, cudaStreamNonBlocking));
            B2_CUDA(cudaStreamCreateWithFlags(&io.d2h, cudaStreamNonBlocking));
            for (int b = 0; b < 2; ++b)
                for (cudaEvent_t* e : {&io.ev_x[b], &io.ev_in[b], &io.ev_fwd[b], &io.ev_bwd[b], &io.ev_out[b]})
                    B2_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
        }
    }
    if (!io.warned_pageable) {
        for (const void* hp : {x_host, dout_host, (const void*)out_host, (const void*)dx_host})
            if (!async_copy_ok(hp)) {
                fprintf(stderr, "b2_moe_fwd_bwd_host: a host buffer is pageable; its copies run synchronously "
                                "and serialise the copy/compute pipeline (use page-locked memory)\n");
                io.warned_pageable = true;
                break;
            }
    }
    const int b = io.next;
    io.next ^= 1;
    char* base = io.dev + (size_t)b * io.slot_bytes;
    void *xd = base, *outd = base + tok_bytes, *doutd = base + 2 * tok_bytes, *dxd = base + 3 * tok_bytes;
    float* auxg = (float*)(base + 4 * tok_bytes);
    cudaStream_t st = cx.stream;
    // inputs: the slot's previous step must be done reading x / dout
    if (io.used[b]) B2_CUDA(cudaStreamWaitEvent(io.h2d, io.ev_bwd[b], 0));
    // the forward waits for x only; dout lands while it runs (the backward waits for it)
    B2_CUDA(cudaMemcpyAsync(xd, x_host, tok_bytes, cudaMemcpyHostToDevice, io.h2d));
    B2_CUDA(cudaEventRecord(io.ev_x[b], io.h2d));
    B2_CUDA(cudaMemcpyAsync(doutd, dout_host, tok_bytes, cudaMemcpyHostToDevice, io.h2d));
    B2_CUDA(cudaEventRecord(io.ev_in[b], io.h2d));
    B2_CUDA(cudaStreamWaitEvent(st, io.ev_x[b], 0));
    if (io.used[b]) B2_CUDA(cudaStreamWaitEvent(st, io.ev_out[b], 0));  // out/dx of the slot read back
    L.forward(xd, router, gate, up, down, s_tokens, false, outd);
    B2_CUDA(cudaStreamWaitEvent(st, io.ev_in[b], 0));
    B2_CUDA(cudaEventRecord(io.ev_fwd[b], st));
    const float* ag = nullptr;
    if (aux_coeff != 0.0) {
        L.aux_probs_grad(aux_coeff, auxg);
        ag = auxg;
    }
    L.backward(router, gate, up, down, doutd, ag, dxd, drouter, dgate, dup, ddown);
    B2_CUDA(cudaEventRecord(io.ev_bwd[b], st));
    // results stream back while the next step computes
    B2_CUDA(cudaStreamWaitEvent(io.d2h, io.ev_fwd[b], 0));
    B2_CUDA(cudaMemcpyAsync(out_host, outd, tok_bytes, cudaMemcpyDeviceToHost, io.d2h));
    B2_CUDA(cudaStreamWaitEvent(io.d2h, io.ev_bwd[b], 0));
    B2_CUDA(cudaMemcpyAsync(dx_host, dxd, tok_bytes, cudaMemcpyDeviceToHost, io.d2h));
    B2_CUDA(cudaEventRecord(io.ev_out[b], io.d2h));
    io.used[b] = true;
}

int b2_moe_fwd_bwd_host(b2_moe* m, const void* x_host, const void* dout_host, const void* router, const void* gate,
                        const void* up, const void* down, double aux_coeff, void* out_host, void* dx_host,
                        void* drouter, void* dgate, void* dup, void* ddown, int64_t s_tokens) {
    return guard([&] {
        fwd_bwd_host_enqueue(m, x_host, dout_host, router, gate, up, down, aux_coeff, out_host, dx_host, drouter,
                             dgate, dup, ddown, s_tokens);
        B2_CUDA(cudaStreamSynchronize(m->io.d2h));
        B2_CUDA(cudaStreamSynchronize(m->ctx->c.stream));
    });
}

int b2_moe_fwd_bwd_host_async(b2_moe* m, const void* x_host, const void* dout_host, const void* router,
                              const void* gate, const void* up, const void* down, double aux_coeff, void* out_host,
                              void* dx_host, void* drouter, void* dgate, void* dup, void* ddown, int64_t s_tokens) {
    return guard([&] {
        fwd_bwd_host_enqueue(m, x_host, dout_host, router, gate, up, down, aux_coeff, out_host, dx_host, drouter,
                             dgate, dup, ddown, s_tokens);
    });
}

int b2_moe_host_wait(b2_moe* m) {
    return guard([&] {
        if (m->io.d2h) B2_CUDA(cudaStreamSynchronize(m->io.d2h));
        if (m->io.h2d) B2_CUDA(cudaStreamSynchronize(m->io.h2d));
        B2_CUDA(cudaStreamSynchronize(m->ctx->c.stream));
    });
}

int b2_route(b2_ctx* ctx, const b2_moe_cfg* cfg, int dtype, const void* x, const void* router, int64_t s_tokens,
             float* logits, float* probs, float* weights, int32_t* indices) {
    return guard([&] {
        MoeConfig c = to_cfg(cfg);
        c.validate();
        cudaStream_t st = ctx->c.stream;
        const int S = (int)s_tokens, H = (int)c.hidden, N = (int)c.n_experts, K = (int)c.top_k;
        if (dtype == F32) launch_router_logits<float>((const float*)x, (const float*)router, logits, S, H, N, st);
        else launch_router_logits<__nv_bfloat16>((const __nv_bfloat16*)x, (const __nv_bfloat16*)router, logits, S, H, N, st);
        launch_softmax_topk(logits, probs, weights, indices, S, N, K, c.normalize_topk, st);
    });
}

int b2_softmax_topk(b2_ctx* ctx, const float* logits, int64_t rows, int64_t n, int64_t k, int normalize, float* probs,
                    float* weights, int32_t* indices) {
    return guard([&] {
        check(k >= 1 && k <= n, "topk: k out of range for width");
        launch_softmax_topk(logits, probs, weights, indices, (int)rows, (int)n, (int)k, normalize != 0, ctx->c.stream);
    });
}

int b2_routing_artifacts(b2_ctx* ctx, const b2_moe_cfg* cfg, const int32_t* indices, int64_t t_total, int ep_rank,
                         int64_t* sizes_host, int64_t* token_counts, int64_t* partial_token_counts,
                         int64_t* partial_cum, int64_t* cum_token_counts, int64_t* expert_counts,
                         int64_t* cum_expert_counts, int64_t* input_indices, int64_t* output_indices,
                         int64_t* selected_k, int64_t* counter) {
    return guard([&] {
        MoeConfig c = to_cfg(cfg);
        c.validate();
        check(ep_rank >= 0 && ep_rank < c.ep, "count_tokens: ep_rank out of range");
        cudaStream_t st = ctx->c.stream;
        const int64_t nr = c.experts_per_rank(), K = c.top_k;
        const int64_t th = ceil_div(t_total, c.token_block);
        const int64_t pmax = round_up(t_total * K + nr * (kRowAlign - 1), kRowAlign);
        const int64_t nch = ceil_div(std::max<int64_t>(t_total, 1), 64);
        Arena ar;
        ar.reserve(4 * (size_t)(2 * nch * nr + 2 * t_total + 2 * nr * th + 3 * nr + 4 * t_total * K + pmax + 64) +
                   32 * 256);
        RoutingIndexArgs a{};
        a.gidx = indices;
        a.T = (int)t_total;
        a.K = (int)K;
        a.N = (int)c.n_experts;
        a.n_start = ep_rank * (int)nr;
        a.nr = (int)nr;
        a.whist = ar.take<int32_t>(nch * nr);
        a.wbase = ar.take<int32_t>(nch * nr);
        a.expert_counts = ar.take<int32_t>(t_total);
        a.cum_expert_counts = ar.take<int32_t>(t_total + 1);
        int32_t* partial_counts = ar.take<int32_t>(nr * th);
        int32_t* partial_cum_d = ar.take<int32_t>(nr * th + 1);
        a.token_counts = ar.take<int32_t>(nr);
        a.cum_token_counts = ar.take<int32_t>(nr + 1);
        a.pad_start = ar.take<int32_t>(nr + 1);
        a.input_indices = ar.take<int32_t>(t_total * K);
        a.output_indices = ar.take<int32_t>(t_total * K);
        a.selected_k = ar.take<int32_t>(t_total * K);
        a.slot_prow = ar.take<int32_t>(t_total * K);
        a.prow_src = ar.take<int32_t>(pmax);
        a.err = ar.take<int32_t>(1);
        B2_CUDA(cudaMemsetAsync(a.err, 0, 4, st));
        launch_routing_index(a, st);
        launch_partial_counts(indices, (int)t_total, (int)K, a.n_start, (int)nr, (int)c.token_block, (int)th,
                              partial_counts, partial_cum_d, st);
        int32_t err = 0;
        B2_CUDA(cudaMemcpyAsync(&err, a.err, 4, cudaMemcpyDeviceToHost, st));
        B2_CUDA(cudaStreamSynchronize(st));
        check(err == 0, "count_tokens: expert id out of range [0," + std::to_string(c.n_experts) + ")");
        auto d2h = [&](const int32_t* d, int64_t n) {
            std::vector<int32_t> t((size_t)std::max<int64_t>(n, 0));
            if (n > 0) B2_CUDA(cudaMemcpy(t.data(), d, 4 * (size_t)n, cudaMemcpyDeviceToHost));
            return std::vector<int64_t>(t.begin(), t.end());
        };
        MoeLayer::HostArtifacts h;
        h.t_total = t_total;
        h.th = th;
        h.cum_token_counts = d2h(a.cum_token_counts, nr + 1);
        h.rt = h.cum_token_counts[(size_t)nr];
        h.pad_start = d2h(a.pad_start, nr + 1);
        h.padded_rows = h.pad_start[(size_t)nr];
        h.token_counts = d2h(a.token_counts, nr);
        h.partial_token_counts = d2h(partial_counts, nr * th);
        h.partial_cum = d2h(partial_cum_d, nr * th + 1);
        h.expert_counts = d2h(a.expert_counts, t_total);
        h.cum_expert_counts = d2h(a.cum_expert_counts, t_total + 1);
        h.input_indices = d2h(a.input_indices, h.rt);
        h.output_indices = d2h(a.output_indices, h.rt);
        h.selected_k = d2h(a.selected_k, h.rt);
        h.counter.resize((size_t)(nr * th));
        for (int64_t i = 0; i < nr * th; ++i) h.counter[(size_t)i] = h.partial_cum[(size_t)i + 1];
        copy_artifacts(h, sizes_host, token_counts, partial_token_counts, partial_cum, cum_token_counts, expert_counts,
                       cum_expert_counts, input_indices, output_indices, selected_k, counter);
    });
}

int b2_opt_create(b2_ctx* ctx, const b2_adamw_cfg* cfg, const b2_param* params, int nparams, int mode,
                  int weight_dtype, int grad_dtype, b2_opt** out) {
    return guard([&] {
        check(ctx != nullptr, "optimizer: null context");
        if (mode < 0 || mode > 2) throw ConfigError("unknown optimizer sharding mode (expected ddp, so, or epso)");
        std::vector<ParamSlot> slots((size_t)nparams);
        for (int i = 0; i < nparams; ++i) {
            slots[(size_t)i].weight = params[i].weight;
            slots[(size_t)i].grad = params[i].grad;
            slots[(size_t)i].numel = params[i].numel;
            slots[(size_t)i].expert = params[i].cls == 1;
            slots[(size_t)i].tp_sharded = params[i].tp_sharded != 0;
        }
        auto o = std::make_unique<b2_opt>();
        o->ctx = ctx;
        o->opt = std::make_unique<ShardedOptimizer>(ctx->c, to_acfg(cfg), std::move(slots), (ShardMode)mode,
                                                    weight_dtype, grad_dtype);
        *out = o.release();
    });
}

int b2_opt_destroy(b2_opt* o) {
    return guard([&] {
        if (!o) return;
        cudaStreamSynchronize(o->ctx->c.stream);
        delete o;
    });
}

int b2_opt_step(b2_opt* o, b2_step_stats* stats) {
    return guard([&] {
        StepStats s = o->opt->step(stats != nullptr);
        if (stats) {
            stats->step = s.step;
            stats->lr = s.lr;
            stats->grad_norm = s.grad_norm;
            stats->clip_scale = s.clip_scale;
            stats->nonfinite = s.nonfinite;
        }
    });
}

int b2_opt_detect_soft_failure(b2_opt* o, double loss, int node, int* sick) {
    return guard([&] { *sick = o->opt->detect_soft_failure(loss, node); });
}

int64_t b2_opt_state_bytes(b2_opt* o) { return o ? o->opt->state_bytes() : -1; }

int b2_opt_owned(b2_opt* o, int p, int64_t* begin, int64_t* end) {
    return guard([&] { o->opt->owned(p, begin, end); });
}

int b2_opt_gather_state(b2_opt* o, int p, float* master, float* exp_avg, float* exp_avg_sq) {
    return guard([&] { o->opt->gather_state(p, master, exp_avg, exp_avg_sq); });
}

int b2_opt_load_state(b2_opt* o, int p, const float* master, const float* exp_avg, const float* exp_avg_sq) {
    return guard([&] { o->opt->load_state(p, master, exp_avg, exp_avg_sq); });
}

int b2_crc32(b2_ctx* ctx, const void* dev, int64_t n, uint32_t crc_in, uint32_t* crc_out) {
    return guard([&] {
        check(ctx && crc_out, "crc32: null argument");
        B2_CUDA(cudaSetDevice(ctx->c.device));
        *crc_out = crc32_device(dev, n, crc_in, ctx->c.stream);
    });
}

int b2_rec_writer_open(b2_ctx* ctx, const char* path, b2_rec_writer** out) {
    return guard([&] {
        check(ctx && path && out, "record writer: null argument");
        require_device();
        *out = reinterpret_cast<b2_rec_writer*>(new RecordWriter(ctx->c.device, ctx->c.stream, path));
    });
}

int b2_rec_writer_add(b2_rec_writer* w, const char* name, int rec_dtype, const int64_t* dims, int ndim,
                      const void* src, int src_dtype) {
    return guard([&] {
        check(w && name && (ndim == 0 || dims) && ndim >= 0, "record writer: null argument");
        check(rec_dtype == B2_REC_F32 || rec_dtype == B2_REC_BF16, "record writer: unknown record dtype");
        reinterpret_cast<RecordWriter*>(w)->add(name, (RecDtype)rec_dtype, std::vector<int64_t>(dims, dims + ndim),
                                                src, src_dtype);
    });
}

int b2_rec_writer_finish(b2_rec_writer* w, int64_t* bytes, uint32_t* crc) {
    std::unique_ptr<RecordWriter> owned(reinterpret_cast<RecordWriter*>(w));
    return guard([&] {
        check(w != nullptr, "record writer: null handle");
        const RecordWriter::Written d = owned->finish();
        if (bytes) *bytes = d.bytes;
        if (crc) *crc = d.crc;
    });
}

int b2_rec_file_open(b2_ctx* ctx, const char* path, b2_rec_file** out) {
    return guard([&] {
        check(ctx && path && out, "record file: null argument");
        require_device();
        *out = reinterpret_cast<b2_rec_file*>(new RecordFile(ctx->c.device, ctx->c.stream, path));
    });
}

int b2_rec_file_count(b2_rec_file* f, int* count) {
    return guard([&] { *count = (int)reinterpret_cast<RecordFile*>(f)->records().size(); });
}

int b2_rec_file_info(b2_rec_file* f, int i, char* name, int name_cap, int* rec_dtype, int64_t* dims, int* ndim) {
    return guard([&] {
        const auto& recs = reinterpret_cast<RecordFile*>(f)->records();
        check(i >= 0 && i < (int)recs.size(), "record file: record index out of range");
        const RecordInfo& r = recs[(size_t)i];
        if (name && name_cap > 0) {
            const size_t k = std::min(r.name.size(), (size_t)name_cap - 1);
            std::memcpy(name, r.name.data(), k);
            name[k] = 0;
        }
        if (rec_dtype) *rec_dtype = (int)r.dtype;
        if (dims)
            for (size_t d = 0; d < r.dims.size(); ++d) dims[d] = r.dims[d];
        if (ndim) *ndim = (int)r.dims.size();
    });
}

int b2_rec_file_find(b2_rec_file* f, const char* name, int* index) {
    return guard([&] { *index = reinterpret_cast<RecordFile*>(f)->find(name); });
}

int b2_rec_file_read(b2_rec_file* f, int i, int64_t begin, int64_t end, void* dst, int dst_dtype) {
    return guard([&] { reinterpret_cast<RecordFile*>(f)->read(i, begin, end, dst, dst_dtype); });
}

int b2_rec_file_close(b2_rec_file* f) {
    return guard([&] { delete reinterpret_cast<RecordFile*>(f); });
}

namespace {
void shard_args(b2_opt* o, const char* const* names, const int64_t* dims, const int* ndims,
                std::vector<std::string>* nm, std::vector<std::vector<int64_t>>* dv) {
    check(o && names, "checkpoint: null argument");
    const int np = o->opt->num_params();
    size_t at = 0;
    for (int p = 0; p < np; ++p) {
        check(names[p] != nullptr, "checkpoint: null parameter name");
        nm->push_back(names[p]);
        std::vector<int64_t> d;
        if (dims && ndims) {
            check(ndims[p] >= 0 && ndims[p] <= 8, "checkpoint: at most 8 dimensions");
            d.assign(dims + at, dims + at + ndims[p]);
            at += (size_t)ndims[p];
        }
        dv->push_back(std::move(d));
    }
}
}  // namespace

int b2_opt_write_shard(b2_opt* o, const char* dir, const char* const* names, const int64_t* dims,
                       const int* ndims, int full, int64_t* bytes, uint32_t* crc, int* model_shard) {
    return guard([&] {
        check(dir != nullptr, "checkpoint: null directory");
        std::vector<std::string> nm;
        std::vector<std::vector<int64_t>> dv;
        shard_args(o, names, dims, ndims, &nm, &dv);
        const ShardWritten w = write_state_shard(*o->opt, dir, nm, dv, full != 0);
        if (bytes) *bytes = w.bytes;
        if (crc) *crc = w.crc;
        if (model_shard) *model_shard = w.model_shard;
    });
}

int b2_opt_restore_shard(b2_opt* o, const char* dir, const char* const* names, const int64_t* dims,
                         const int* ndims, int full) {
    return guard([&] {
        check(dir != nullptr, "checkpoint: null directory");
        std::vector<std::string> nm;
        std::vector<std::vector<int64_t>> dv;
        shard_args(o, names, dims, ndims, &nm, &dv);
        restore_state_shard(*o->opt, dir, nm, dv, full != 0);
    });
}

int b2_opt_get_state(b2_opt* o, int p, float* master, float* exp_avg, float* exp_avg_sq) {
    return guard([&] { o->opt->get_state(p, master, exp_avg, exp_avg_sq); });
}

int b2_opt_set_step_count(b2_opt* o, int64_t n) {
    return guard([&] { o->opt->set_step_count(n); });
}

int b2_adamw_update(b2_ctx* ctx, float* master, float* exp_avg, float* exp_avg_sq, const void* grad, int grad_dtype,
                    int64_t n, double lr, int64_t step, const b2_adamw_cfg* cfg, void* weight_out, int weight_dtype,
                    int round_bf16) {
    return guard([&] {
        AdamWConfig c = to_acfg(cfg);
        AdamWKernelArgs a{};
        a.master = master;
        a.m = exp_avg;
        a.v = exp_avg_sq;
        a.grad = grad;
        a.weight_out = weight_out;
        a.n = n;
        a.grad_dtype = grad_dtype;
        a.weight_dtype = weight_dtype;
        a.lr = lr;
        a.beta1 = c.beta1;
        a.beta2 = c.beta2;
        a.eps = c.eps;
        a.weight_decay = c.weight_decay;
        a.bc1 = 1.0 - std::pow(c.beta1, (double)(step + 1));
        a.bc2 = 1.0 - std::pow(c.beta2, (double)(step + 1));
        a.grad_scale = 1.0;
        a.round_bf16 = round_bf16;
        launch_adamw(a, ctx->c.stream);
    });
}

double b2_lr_at_step(int64_t step, const b2_adamw_cfg* cfg) {
    double r = -1.0;
    guard([&] { r = lr_at_step(step, to_acfg(cfg)); });
    return r;
}

int b2_memory_report(int64_t p_expert, int64_t p_non_expert, int mode, int dp, int ep, double capacity_gb,
                     b2_memory_report_t* out) {
    return guard([&] {
        check(out != nullptr, "memory_report: null output");
        const MemoryReport r = memory_report(p_expert, p_non_expert, mode, dp, ep, capacity_gb);
        out->weights_bytes = r.weights_bytes;
        out->grads_bytes = r.grads_bytes;
        out->master_bytes = r.master_bytes;
        out->optim_bytes = r.optim_bytes;
        out->total_bytes = r.total_bytes;
        out->capacity_bytes = r.capacity_bytes;
        out->feasible = r.feasible ? 1 : 0;
    });
}

int b2_shard_slice(int64_t numel, int group_size, int position, int64_t* begin, int64_t* end) {
    return guard([&] { shard_slice(numel, group_size, position, begin, end); });
}

int b2_moe_set_profiling(b2_moe* m, int on) { return guard([&] { m->layer->set_profiling(on); }); }
int b2_moe_set_graph(b2_moe* m, int on) { return guard([&] { m->layer->set_graph(on != 0); }); }
int b2_moe_stage_times(b2_moe* m, float* ms_host) { return guard([&] { m->layer->stage_times(ms_host); }); }
const char* b2_moe_stage_name(int stage) { return MoeLayer::stage_name(stage); }

int b2_moe_last_launches(b2_moe* m) { return m ? m->layer->last_launches() : 0; }
int b2_opt_last_launches(b2_opt* o) { return o ? o->opt->last_launches() : 0; }

}  // extern "C"

#include "../../include/b2moe_testing.h"

extern "C" int b2x_moe_set_overlap_return(b2_moe* m, int on) {
    return guard([&] { m->layer->set_overlap_return(on != 0); });
}

extern "C" int b2x_grouped_gemm(b2_ctx* ctx, int kind, int hidden, int intermediate, int nr, const int32_t* pad_start,
                                const int32_t* counts, int64_t pmax, const void* x, const void* wg, const void* wu, const void* wd,
                                const void* g, const void* u, const void* h, const void* dy, const void* dgu,
                                void* out0, void* out1, void* out2, float scale) {
    return guard([&] {
        check(kind >= 0 && kind <= 5, "grouped gemm: unknown kind");
        check(sm100_available(), "tcgen05 grouped GEMM needs an sm_100 (B200) device");
        Sm100GemmArgs a{};
        a.kind = (GemmKind)kind;
        a.H = hidden;
        a.I = intermediate;
        a.nr = nr;
        a.pmax = pmax;
        a.pad_start = pad_start;
        a.counts = counts;
        a.x = x;
        a.wg = wg;
        a.wu = wu;
        a.wd = wd;
        a.g = g;
        a.u = u;
        a.h = h;
        a.dy = dy;
        a.dgu = dgu;
        a.out0 = out0;
        a.out1 = out1;
        a.out2 = out2;
        a.scale = scale;
        a.num_sms = ctx->c.num_sms;
        launch_sm100_gemm(a, ctx->c.stream);
    });
}
