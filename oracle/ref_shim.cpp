// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// extern "C" shim over the UNMODIFIED reference implementation
// (/root/reference/proj, compiled in place by oracle/Makefile into
// oracle/_ref/libref_optimus.so). It exposes the reference's own hot-path
// functions to the parity tests and to bench.py's cpu_baseline / --impl
// reference arm:
//   route                  include/optimus/moe.hpp:58-80
//   count_tokens           include/optimus/moe.hpp:122-164
//   generate_indices       include/optimus/moe.hpp:167-197
//   fast_moe_forward       include/optimus/moe.hpp:344-390
//   fast_moe_backward      include/optimus/moe.hpp:392-466
//   moe_aux_probs_grad     include/optimus/moe.hpp:331-342
//   reference_moe_forward  include/optimus/moe.hpp:471-497 (dense per-token oracle)
//   adamw_update           src/optim.cpp:88-107
//   lr_at_step             src/optim.cpp:17-24
//   shard_slice            src/optim.cpp:43-50
//   memory_report          src/optim.cpp:196-221
//   ShardedOptimizer::step src/optim.cpp:130-194
//   Model::param_slots     src/model.cpp:189-229 (the EPSO parameter set of bench.py)
//   count_params / preset  src/model.cpp:31-91
// The rank threads are the reference's own World (src/comm.cpp:80-124).
#include <chrono>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "optimus/comm.hpp"
#include "optimus/model.hpp"
#include "optimus/moe.hpp"
#include "optimus/optim.hpp"

using namespace optimus;

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const ContractError& e) {
        g_err = e.what();
        return 1;
    } catch (const ConfigError& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 9;
    }
}
}  // namespace

extern "C" {

struct ref_moe_cfg {
    int64_t n_experts, top_k, hidden, intermediate;
    int32_t ep;
    int32_t normalize_topk;
    int64_t token_block;
};

const char* ref_last_error() { return g_err.c_str(); }

static MoeConfig to_cfg(const ref_moe_cfg* c) {
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

int ref_route_f32(const ref_moe_cfg* c, int64_t s, const float* x, const float* router,
                  float* logits, float* probs, float* weights, int64_t* indices) {
    return guard([&] {
        MoeConfig cfg = to_cfg(c);
        TensorF xt({s, cfg.hidden}, std::vector<float>(x, x + s * cfg.hidden));
        TensorF rt({cfg.hidden, cfg.n_experts},
                   std::vector<float>(router, router + cfg.hidden * cfg.n_experts));
        RouteResult<float> r = route(xt, rt, cfg);
        std::memcpy(logits, r.logits.data(), r.logits.bytes());
        std::memcpy(probs, r.probs.data(), r.probs.bytes());
        std::memcpy(weights, r.weights.data(), r.weights.bytes());
        std::memcpy(indices, r.indices.data(), r.indices.bytes());
    });
}

// softmax / topk on caller-provided scores (kernels.hpp:194-258)
int ref_softmax_topk_f32(int64_t rows, int64_t n, int64_t k, const float* logits, float* probs,
                         float* values, int64_t* indices) {
    return guard([&] {
        TensorF lt({rows, n}, std::vector<float>(logits, logits + rows * n));
        TensorF p = softmax(lt);
        std::memcpy(probs, p.data(), p.bytes());
        auto [v, i] = topk(p, k);
        std::memcpy(values, v.data(), v.bytes());
        std::memcpy(indices, i.data(), i.bytes());
    });
}

// Every output buffer is caller-sized for the maxima: partial_* hold NR*TH(+1),
// rt-sized arrays hold T*K. out_sizes = {th, rt}.
int ref_routing_artifacts(const ref_moe_cfg* c, int64_t t_total, const int64_t* indices,
                          int ep_rank, int64_t* out_sizes, int64_t* token_counts,
                          int64_t* partial_token_counts, int64_t* partial_cum,
                          int64_t* cum_token_counts, int64_t* expert_counts,
                          int64_t* cum_expert_counts, int64_t* input_indices,
                          int64_t* output_indices, int64_t* selected_k, int64_t* counter) {
    return guard([&] {
        MoeConfig cfg = to_cfg(c);
        TensorI idx({t_total, cfg.top_k}, std::vector<int64_t>(indices, indices + t_total * cfg.top_k));
        RoutingArtifacts a = count_tokens(idx, ep_rank, cfg);
        generate_indices(idx, ep_rank, cfg, a);
        out_sizes[0] = a.th;
        out_sizes[1] = a.rt;
        auto cp = [](int64_t* dst, const TensorI& t) {
            if (dst && t.numel()) std::memcpy(dst, t.data(), t.bytes());
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
    });
}

// One MoE layer forward (+ optional backward) on an EP world of cfg->ep rank
// threads. Inputs are the FULL logical tensors: x_full/dout_full [EP*S, H],
// router [H, N], gate/up [N, H, I], down [N, I, H]; each rank takes its S-row
// slice and its NR-expert block, exactly like the reference tests do
// (test_moe.cpp:645-716). Outputs are assembled back into full tensors:
//   out/dx [EP*S,H], weights/idx/probs for the local rows [EP*S,*],
//   drouter [EP, H, N] (per-rank partials), dgate/dup/ddown [N,...] (already
//   scaled by 1/EP as the reference does), aux [EP].
}  // extern "C"
template <typename T>
static int moe_layer_impl(const ref_moe_cfg* c, int64_t s_local, const T* x_full,
                          const T* router, const T* gate_full, const T* up_full,
                          const T* down_full, const T* dout_full, int fur, double aux_coeff,
                          int do_backward, T* out_full, T* dx_full, T* drouter, T* dgate,
                          T* dup, T* ddown, T* weights_out, int64_t* idx_out, T* probs_out,
                          double* aux_out) {
    return guard([&] {
        MoeConfig cfg = to_cfg(c);
        cfg.validate();
        const int64_t H = cfg.hidden, I = cfg.intermediate, N = cfg.n_experts, K = cfg.top_k;
        const int64_t NR = cfg.experts_per_rank();
        Topology topo;
        topo.ep = cfg.ep;
        World world(topo);
        world.run([&](RankCtx& ctx) {
            const int er = ctx.coord().ep;
            ExpertWeights<T> w;
            w.router = Tensor<T>({H, N}, std::vector<T>(router, router + H * N));
            const int64_t blk = H * I;
            w.gate = Tensor<T>({NR, H, I}, std::vector<T>(gate_full + er * NR * blk,
                                                           gate_full + (er + 1) * NR * blk));
            w.up = Tensor<T>({NR, H, I}, std::vector<T>(up_full + er * NR * blk,
                                                         up_full + (er + 1) * NR * blk));
            w.down = Tensor<T>({NR, I, H}, std::vector<T>(down_full + er * NR * blk,
                                                           down_full + (er + 1) * NR * blk));
            Tensor<T> x({s_local, H}, std::vector<T>(x_full + er * s_local * H,
                                                      x_full + (er + 1) * s_local * H));
            FastMoeState<T> st;
            Tensor<T> out = fast_moe_forward<T>(ctx, ctx.ep_group(), x, w, cfg, fur != 0, &st);
            std::memcpy(out_full + er * s_local * H, out.data(), out.bytes());
            if (weights_out)
                std::memcpy(weights_out + er * s_local * K, st.routing.weights.data(),
                            st.routing.weights.bytes());
            if (idx_out)
                std::memcpy(idx_out + er * s_local * K, st.routing.indices.data(),
                            st.routing.indices.bytes());
            if (probs_out)
                std::memcpy(probs_out + er * s_local * N, st.routing.probs.data(),
                            st.routing.probs.bytes());
            if (aux_out) aux_out[er] = moe_aux_loss(st);
            if (!do_backward) return;
            Tensor<T> dout({s_local, H}, std::vector<T>(dout_full + er * s_local * H,
                                                         dout_full + (er + 1) * s_local * H));
            Tensor<T> apg;
            const Tensor<T>* apg_ptr = nullptr;
            if (aux_coeff != 0.0) {
                apg = moe_aux_probs_grad<T>(st, aux_coeff);
                apg_ptr = &apg;
            }
            MoeGrads<T> g = fast_moe_backward<T>(ctx, ctx.ep_group(), st, w, dout, apg_ptr);
            std::memcpy(dx_full + er * s_local * H, g.input.data(), g.input.bytes());
            std::memcpy(drouter + er * H * N, g.router.data(), g.router.bytes());
            std::memcpy(dgate + er * NR * blk, g.gate.data(), g.gate.bytes());
            std::memcpy(dup + er * NR * blk, g.up.data(), g.up.bytes());
            std::memcpy(ddown + er * NR * blk, g.down.data(), g.down.bytes());
        });
    });
}

extern "C" {
// reference_moe_forward (include/optimus/moe.hpp:471-497): the dense per-token oracle over the
// full expert set; weights/indices are the routing of the same tokens ([T,K]).
int ref_dense_moe_forward_f32(const ref_moe_cfg* c, int64_t t_total, const float* x,
                              const float* gate, const float* up, const float* down,
                              const float* weights, const int64_t* indices, float* out) {
    return guard([&] {
        MoeConfig cfg = to_cfg(c);
        cfg.validate();
        const int64_t H = cfg.hidden, I = cfg.intermediate, N = cfg.n_experts, K = cfg.top_k;
        ExpertWeights<float> w;
        w.gate = Tensor<float>({N, H, I}, std::vector<float>(gate, gate + N * H * I));
        w.up = Tensor<float>({N, H, I}, std::vector<float>(up, up + N * H * I));
        w.down = Tensor<float>({N, I, H}, std::vector<float>(down, down + N * I * H));
        Tensor<float> in({t_total, H}, std::vector<float>(x, x + t_total * H));
        Tensor<float> wt({t_total, K}, std::vector<float>(weights, weights + t_total * K));
        TensorI idx({t_total, K}, std::vector<int64_t>(indices, indices + t_total * K));
        Tensor<float> o = reference_moe_forward<float>(in, w, wt, idx, cfg);
        std::memcpy(out, o.data(), o.bytes());
    });
}
}  // extern "C"

extern "C" {
int ref_moe_layer_f32(const ref_moe_cfg* c, int64_t s_local, const float* x, const float* router,
                      const float* gate, const float* up, const float* down, const float* dout,
                      int fur, double aux_coeff, int do_backward, float* out, float* dx,
                      float* drouter, float* dgate, float* dup, float* ddown, float* weights,
                      int64_t* idx, float* probs, double* aux) {
    return moe_layer_impl<float>(c, s_local, x, router, gate, up, down, dout, fur, aux_coeff,
                                 do_backward, out, dx, drouter, dgate, dup, ddown, weights, idx,
                                 probs, aux);
}

int ref_moe_layer_f64(const ref_moe_cfg* c, int64_t s_local, const double* x,
                      const double* router, const double* gate, const double* up,
                      const double* down, const double* dout, int fur, double aux_coeff,
                      int do_backward, double* out, double* dx, double* drouter, double* dgate,
                      double* dup, double* ddown, double* weights, int64_t* idx, double* probs,
                      double* aux) {
    return moe_layer_impl<double>(c, s_local, x, router, gate, up, down, dout, fur, aux_coeff,
                                  do_backward, out, dx, drouter, dgate, dup, ddown, weights, idx,
                                  probs, aux);
}

// the reference's deterministic generators (common.hpp:83-87, kernels.hpp:392-399,
// moe.hpp:500-523): used to produce the exact synthetic inputs of SURVEY §8d
void ref_normal_init_f32(float* out, int64_t n, uint64_t seed, uint64_t tag, double stddev) {
    for (int64_t i = 0; i < n; ++i) out[i] = (float)(normal_at(seed, tag, (uint64_t)i) * stddev);
}
uint64_t ref_fnv1a(const char* s) { return fnv1a(s); }
uint64_t ref_hash_mix(uint64_t a, uint64_t b) { return hash_mix(a, b); }
float ref_bf16_round(float f) { return bf16_round(f); }

// ---- optimizer ------------------------------------------------------------------------

struct ref_adamw_cfg {
    double beta1, beta2, eps, weight_decay, peak_lr, min_lr;
    int64_t warmup_steps, total_steps;
    double clip_norm;
    int32_t clip_after_warmup_only, round_weights_bf16;
};

static AdamWConfig to_acfg(const ref_adamw_cfg* a) {
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

void ref_adamw_default_cfg(ref_adamw_cfg* out) {
    AdamWConfig c;
    out->beta1 = c.beta1;
    out->beta2 = c.beta2;
    out->eps = c.eps;
    out->weight_decay = c.weight_decay;
    out->peak_lr = c.peak_lr;
    out->min_lr = c.min_lr;
    out->warmup_steps = c.warmup_steps;
    out->total_steps = c.total_steps;
    out->clip_norm = c.clip_norm;
    out->clip_after_warmup_only = c.clip_after_warmup_only;
    out->round_weights_bf16 = c.round_weights_bf16;
}

double ref_lr_at_step(int64_t step, const ref_adamw_cfg* a) { return lr_at_step(step, to_acfg(a)); }

int ref_memory_report(int64_t p_expert, int64_t p_non_expert, int mode, int dp, int ep, double capacity_gb,
                      double* out) {
    return guard([&] {
        const MemoryReport r = memory_report(p_expert, p_non_expert, (ShardMode)mode, dp, ep, capacity_gb);
        const double v[7] = {r.weights_bytes, r.grads_bytes, r.master_bytes, r.optim_bytes,
                             r.total_bytes,   r.capacity_bytes, r.feasible ? 1.0 : 0.0};
        std::memcpy(out, v, sizeof(v));
    });
}

int ref_shard_slice(int64_t numel, int g, int pos, int64_t* begin, int64_t* end) {
    return guard([&] {
        SliceRange r = shard_slice(numel, g, pos);
        *begin = r.begin;
        *end = r.end;
    });
}

int ref_adamw_update(float* master, float* m, float* v, const float* grad, int64_t n, double lr,
                     int64_t step, const ref_adamw_cfg* a, float* weight_out, int round_bf16) {
    return guard([&] {
        AdamWState st;
        st.master.assign(master, master + n);
        st.exp_avg.assign(m, m + n);
        st.exp_avg_sq.assign(v, v + n);
        adamw_update(st, grad, n, lr, step, to_acfg(a), weight_out, round_bf16 != 0);
        std::memcpy(master, st.master.data(), (size_t)n * 4);
        std::memcpy(m, st.exp_avg.data(), (size_t)n * 4);
        std::memcpy(v, st.exp_avg_sq.data(), (size_t)n * 4);
    });
}

// Runs ShardedOptimizer::step `steps` times on a dp x ep (x tp) world.
//   numel[p], cls[p] (0 non_expert, 1 expert), tp_sharded[p]
//   w_init: per rank, all params concatenated (rank-major, world_size * total)
//   grads:  per step, per rank, all params concatenated
//   w_out:  final weights per rank (same layout as w_init)
//   master_out/m_out/v_out: per rank, owned slices concatenated in param order
//     (caller-sized world_size * total; unused tail left untouched)
//   owned_out: per rank per param [begin,end)
//   stats_out: per step per rank {lr, grad_norm, clip_scale}
//   state_bytes_out: per rank
int ref_sharded_steps(int dp, int ep, int tp, int mode, const ref_adamw_cfg* a, int nparams,
                      const int64_t* numel, const int* cls, const int* tp_sharded,
                      const float* w_init, const float* grads, int steps, float* w_out,
                      float* master_out, float* m_out, float* v_out, int64_t* owned_out,
                      double* stats_out, int64_t* state_bytes_out) {
    return guard([&] {
        Topology topo;
        topo.dp = dp;
        topo.ep = ep;
        topo.tp = tp;
        World world(topo);
        const int W = topo.world_size();
        int64_t total = 0;
        for (int p = 0; p < nparams; ++p) total += numel[p];
        world.run([&](RankCtx& ctx) {
            const int r = ctx.rank();
            std::vector<TensorF> ws, gs;
            ws.reserve((size_t)nparams);
            gs.reserve((size_t)nparams);
            int64_t off = 0;
            for (int p = 0; p < nparams; ++p) {
                const float* src = w_init + (int64_t)r * total + off;
                ws.emplace_back(std::vector<int64_t>{numel[p]}, std::vector<float>(src, src + numel[p]));
                gs.emplace_back(std::vector<int64_t>{numel[p]});
                off += numel[p];
            }
            std::vector<ParamSlot> slots;
            for (int p = 0; p < nparams; ++p)
                slots.push_back({strcat_("p", p), &ws[(size_t)p], &gs[(size_t)p],
                                 cls[p] ? ReplicationClass::expert : ReplicationClass::non_expert,
                                 tp_sharded[p] != 0});
            ShardedOptimizer opt(ctx, to_acfg(a), slots, (ShardMode)mode);
            for (int s = 0; s < steps; ++s) {
                int64_t o = 0;
                for (int p = 0; p < nparams; ++p) {
                    const float* src = grads + ((int64_t)s * W + r) * total + o;
                    std::memcpy(gs[(size_t)p].data(), src, (size_t)numel[p] * 4);
                    o += numel[p];
                }
                StepStats st = opt.step();
                double* so = stats_out + ((int64_t)s * W + r) * 3;
                so[0] = st.lr;
                so[1] = st.grad_norm;
                so[2] = st.clip_scale;
            }
            int64_t o = 0, so = 0;
            for (int p = 0; p < nparams; ++p) {
                std::memcpy(w_out + (int64_t)r * total + o, ws[(size_t)p].data(), (size_t)numel[p] * 4);
                o += numel[p];
                const SliceRange own = opt.plan().entries[(size_t)p].own;
                owned_out[((int64_t)r * nparams + p) * 2 + 0] = own.begin;
                owned_out[((int64_t)r * nparams + p) * 2 + 1] = own.end;
                const AdamWState& st = opt.states()[(size_t)p];
                std::memcpy(master_out + (int64_t)r * total + so, st.master.data(), st.master.size() * 4);
                std::memcpy(m_out + (int64_t)r * total + so, st.exp_avg.data(), st.exp_avg.size() * 4);
                std::memcpy(v_out + (int64_t)r * total + so, st.exp_avg_sq.data(), st.exp_avg_sq.size() * 4);
                so += (int64_t)st.master.size();
            }
            state_bytes_out[r] = opt.state_bytes();
        });
    });
}

// ---- CPU baseline timers (bench.py cpu_baseline / --impl reference) -----------------------

// fwd+bwd of one MoE layer on an EP world of `ep` rank threads with s_local tokens
// per rank, reference synthetic inputs; returns seconds per iteration
// (best of iters) via *sec.
int ref_bench_moe_f32(const ref_moe_cfg* c, int64_t s_local, int iters, double* sec) {
    return guard([&] {
        MoeConfig cfg = to_cfg(c);
        cfg.validate();
        const int64_t H = cfg.hidden, N = cfg.n_experts;
        double best = 1e30;
        for (int it = 0; it < iters; ++it) {
            Topology topo;
            topo.ep = cfg.ep;
            World world(topo);
            std::vector<double> per((size_t)cfg.ep, 0.0);
            world.run([&](RankCtx& ctx) {
                const int er = ctx.coord().ep;
                ExpertWeights<float> w = init_expert_weights<float>(cfg, er, 1234, 0.02);
                (void)N;
                TensorF x = normal_init<float>({s_local, H}, 77, (uint64_t)ctx.rank(), 1.0);
                TensorF dout = normal_init<float>({s_local, H}, 78, (uint64_t)ctx.rank(), 1.0);
                barrier(ctx, ctx.ep_group());
                auto t0 = std::chrono::steady_clock::now();
                FastMoeState<float> st;
                fast_moe_forward<float>(ctx, ctx.ep_group(), x, w, cfg, false, &st);
                TensorF apg = moe_aux_probs_grad<float>(st, 0.01);
                MoeGrads<float> g = fast_moe_backward<float>(ctx, ctx.ep_group(), st, w, dout, &apg);
                barrier(ctx, ctx.ep_group());
                auto t1 = std::chrono::steady_clock::now();
                per[(size_t)er] = std::chrono::duration<double>(t1 - t0).count();
            });
            double mx = 0;
            for (double v : per) mx = std::max(mx, v);
            best = std::min(best, mx);
        }
        *sec = best;
    });
}

// ShardedOptimizer::step on a dp x ep world over one synthetic param set of
// n_expert + n_non_expert elements (per rank); seconds per step via *sec
int ref_bench_optim(int dp, int ep, int mode, int64_t n_expert, int64_t n_non_expert, int steps,
                    double* sec) {
    return guard([&] {
        Topology topo;
        topo.dp = dp;
        topo.ep = ep;
        World world(topo);
        std::vector<double> per((size_t)topo.world_size(), 0.0);
        world.run([&](RankCtx& ctx) {
            TensorF we = normal_init<float>({n_expert}, 500, 100 + (uint64_t)ctx.coord().ep, 0.02);
            TensorF wn = normal_init<float>({n_non_expert}, 501, 1, 0.02);
            TensorF ge({n_expert}), gn({n_non_expert});
            std::vector<ParamSlot> slots = {
                {"ne", &wn, &gn, ReplicationClass::non_expert, false},
                {"ex", &we, &ge, ReplicationClass::expert, false},
            };
            AdamWConfig cfg;
            cfg.warmup_steps = 0;
            ShardedOptimizer opt(ctx, cfg, slots, (ShardMode)mode);
            double best = 1e30;
            for (int s = 0; s < steps; ++s) {
                const uint64_t salt = hash_mix((uint64_t)s, (uint64_t)ctx.rank());
                for (int64_t i = 0; i < n_expert; ++i)
                    ge.data()[i] = bf16_round((float)(normal_at(502, salt, (uint64_t)i) * 1e-3));
                for (int64_t i = 0; i < n_non_expert; ++i)
                    gn.data()[i] = bf16_round((float)(normal_at(503, salt, (uint64_t)i) * 1e-3));
                barrier(ctx, ctx.world_group());
                auto t0 = std::chrono::steady_clock::now();
                opt.step();
                barrier(ctx, ctx.world_group());
                auto t1 = std::chrono::steady_clock::now();
                best = std::min(best, std::chrono::duration<double>(t1 - t0).count());
            }
            per[(size_t)ctx.rank()] = best;
        });
        double mx = 0;
        for (double v : per) mx = std::max(mx, v);
        *sec = mx;
    });
}

}  // extern "C"

// ---- record files: RecordFileWriter / read_record_file (src/reliability.cpp:222-320) ----
#include "optimus/reliability.hpp"

extern "C" {
// names NUL-separated; data: every record's f32 values concatenated (add_f32 / add_bf16)
int ref_record_file_write(const char* path, int n_rec, const char* names, const int32_t* dtypes,
                          const int32_t* ndims, const int64_t* dims, const float* data, int64_t* bytes,
                          uint32_t* crc) {
    return guard([&] {
        RecordFileWriter w(path);
        int64_t di = 0, de = 0;
        for (int r = 0; r < n_rec; ++r) {
            const std::string name(names);
            names += name.size() + 1;
            std::vector<int64_t> d(dims + di, dims + di + ndims[r]);
            di += ndims[r];
            int64_t n = 1;
            for (int64_t x : d) n *= x;
            if (dtypes[r] == 0)
                w.add_f32(name, d, data + de, n);
            else
                w.add_bf16(name, d, data + de, n);
            de += n;
        }
        const RecordFileWriter::Written done = w.finish();
        *bytes = done.bytes;
        *crc = done.crc;
    });
}

// read_record_file: count, total elements, and (data_out) every record as_f32, concatenated
int ref_record_file_read(const char* path, int64_t* count, int64_t* total, float* data_out, int64_t cap) {
    return guard([&] {
        std::vector<TensorRecord> recs = read_record_file(path);
        int64_t tot = 0;
        for (const TensorRecord& r : recs) {
            std::vector<float> f = r.as_f32();
            for (size_t e = 0; e < f.size() && data_out; ++e)
                if (tot + (int64_t)e < cap) data_out[tot + (int64_t)e] = f[e];
            tot += (int64_t)f.size();
        }
        *count = (int64_t)recs.size();
        *total = tot;
    });
}
}  // extern "C"

// ---- the model's parameter slots (bench.py's EPSO parameter set is pinned to these) ----------
extern "C" {

// the preset's parameter count (model.cpp:70-91)
int ref_count_params(const char* preset_name, int64_t* total, int64_t* active) {
    return guard([&] {
        const ParamCount pc = count_params(preset(preset_name));
        *total = pc.total;
        *active = pc.active;
    });
}

// Model::param_slots of the rank at EP coordinate ep_coord (Topology{ep}) for a preset;
// writes up to cap slots (numel, expert?, tp_sharded?) and returns the slot count in *n
int ref_param_slots(const char* preset_name, int ep, int ep_coord, int64_t* numel, int32_t* expert, int32_t* tp,
                    int cap, int* n) {
    return guard([&] {
        Topology topo;
        topo.ep = ep;
        RankCoord coord;
        coord.ep = ep_coord;
        Model m(preset(preset_name), topo, coord, 1234);
        const std::vector<ParamSlot> slots = m.param_slots();
        *n = (int)slots.size();
        for (int i = 0; i < (int)slots.size() && i < cap; ++i) {
            numel[i] = slots[(size_t)i].weight->numel();
            expert[i] = slots[(size_t)i].cls == ReplicationClass::expert ? 1 : 0;
            tp[i] = slots[(size_t)i].tp_sharded ? 1 : 0;
        }
    });
}

}  // extern "C"
