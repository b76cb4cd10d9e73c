/* TEST INFRASTRUCTURE ONLY — CPU restatement of the reference hot path, used
 * as the parity checker by tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg. The product library (paper_2604_00785_b200/) never links
 * or calls anything in oracle/.
 *
 * Restated from the reference (file:line under /root/reference/proj):
 *   common.hpp:52-87     splitmix64 / hash_mix / fnv1a / normal_at (input generators)
 *   common.hpp:116-131   bf16 round-to-nearest-even
 *   moe.hpp:13-31        MoeConfig::validate
 *   moe.hpp:122-164      count_tokens
 *   moe.hpp:167-197      generate_indices
 *   moe_oracle_impl.h    route / expert MLP / reductions / backward (moe.hpp:58-466),
 *                        dense per-token reference_moe_forward (moe.hpp:471-497)
 *   optim.cpp:17-24      lr_at_step
 *   optim.cpp:43-50      shard_slice
 *   optim.cpp:196-221    memory_report
 *   optim.cpp:52-86      build_shard_plan / counts_toward_norm
 *   optim.cpp:88-107     adamw_update
 *   optim.cpp:130-194    ShardedOptimizer::step (collectives simulated in member order)
 *
 * Pinned: tests/test_oracle_pin.py checks every entry point bitwise against the
 * reference compiled in place (oracle/_ref/libref_optimus.so) and against the
 * reference's own known-answer tests (tests/golden/). Build: oracle/Makefile. */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    int64_t n_experts, top_k, hidden, intermediate;
    int32_t ep;
    int32_t normalize_topk;
    int64_t token_block;
} orc_moe_cfg;

typedef struct {
    int64_t t_total, th, rt, nr;
    int64_t *token_counts, *partial_token_counts, *partial_cum, *cum_token_counts;
    int64_t *expert_counts, *cum_expert_counts;
    int64_t *input_indices, *output_indices, *selected_k, *counter;
} orc_artifacts;

static char g_err[256];
const char* orc_last_error(void) { return g_err; }

/* ---- generators (common.hpp:52-87) ------------------------------------------------ */

static uint64_t splitmix64(uint64_t* state) {
    uint64_t z = (*state += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
uint64_t orc_hash_mix(uint64_t a, uint64_t b) {
    uint64_t s = a * 0x9e3779b97f4a7c15ull + b;
    return splitmix64(&s);
}
static uint64_t hash_mix3(uint64_t a, uint64_t b, uint64_t c) { return orc_hash_mix(orc_hash_mix(a, b), c); }
uint64_t orc_fnv1a(const char* s) {
    uint64_t h = 0xcbf29ce484222325ull;
    for (const unsigned char* p = (const unsigned char*)s; *p; ++p) {
        h ^= *p;
        h *= 0x100000001b3ull;
    }
    return h;
}
static double u64_to_unit(uint64_t x) { return (double)((x >> 11) + 1) * (1.0 / 9007199254740992.0); }
double orc_normal_at(uint64_t seed, uint64_t tag, uint64_t i) {
    double u1 = u64_to_unit(hash_mix3(seed, tag, 2 * i));
    double u2 = u64_to_unit(hash_mix3(seed, tag, 2 * i + 1));
    return sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
}
void orc_normal_init_f32(float* out, int64_t n, uint64_t seed, uint64_t tag, double stddev) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) out[i] = (float)(orc_normal_at(seed, tag, (uint64_t)i) * stddev);
}
void orc_normal_init_f64(double* out, int64_t n, uint64_t seed, uint64_t tag, double stddev) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) out[i] = orc_normal_at(seed, tag, (uint64_t)i) * stddev;
}
/* rng.next_below used by the reference tests (common.hpp:90-100) */
uint64_t orc_rng_next(uint64_t* state) { return splitmix64(state); }

/* ---- bf16 (common.hpp:116-131) ------------------------------------------------------ */

uint16_t orc_f32_to_bf16_bits(float f) {
    uint32_t u;
    memcpy(&u, &f, 4);
    if (isnan(f)) return (uint16_t)((u >> 16) | 0x0040);
    uint32_t rounded = u + 0x7fffu + ((u >> 16) & 1u);
    return (uint16_t)(rounded >> 16);
}
float orc_bf16_round(float f) {
    uint32_t u = (uint32_t)orc_f32_to_bf16_bits(f) << 16;
    float r;
    memcpy(&r, &u, 4);
    return r;
}
void orc_bf16_round_array(float* x, int64_t n) {
    for (int64_t i = 0; i < n; ++i) x[i] = orc_bf16_round(x[i]);
}

/* ---- config / artifacts (moe.hpp:13-31, 122-197) --------------------------------------- */

static int orc_validate(const orc_moe_cfg* c) {
    if (!(c->n_experts >= 1 && c->top_k >= 1 && c->hidden >= 1 && c->intermediate >= 1 && c->ep >= 1)) {
        strcpy(g_err, "moe: config fields must be positive");
        return 1;
    }
    if (c->top_k > c->n_experts) {
        strcpy(g_err, "moe: top_k cannot exceed n_experts");
        return 1;
    }
    if (c->n_experts % c->ep != 0) {
        strcpy(g_err, "moe: n_experts must divide evenly over ep");
        return 1;
    }
    if (c->token_block < 1) {
        strcpy(g_err, "moe: token_block must be positive");
        return 1;
    }
    return 0;
}
int orc_cfg_validate(const orc_moe_cfg* c) { return orc_validate(c); }

static void orc_artifacts_free(orc_artifacts* a) {
    free(a->token_counts);
    free(a->partial_token_counts);
    free(a->partial_cum);
    free(a->cum_token_counts);
    free(a->expert_counts);
    free(a->cum_expert_counts);
    free(a->input_indices);
    free(a->output_indices);
    free(a->selected_k);
    free(a->counter);
    memset(a, 0, sizeof(*a));
}

static int64_t* zalloc64(int64_t n) { return (int64_t*)calloc((size_t)(n > 0 ? n : 1), 8); }

/* count_tokens (moe.hpp:122-164) followed by generate_indices (moe.hpp:167-197) */
static int orc_artifacts_build(const orc_moe_cfg* c, int64_t t_total, const int64_t* indices,
                               int ep_rank, orc_artifacts* a) {
    if (orc_validate(c)) return 1;
    if (ep_rank < 0 || ep_rank >= c->ep) {
        strcpy(g_err, "count_tokens: ep_rank out of range");
        return 1;
    }
    const int64_t K = c->top_k, nr = c->n_experts / c->ep, tbs = c->token_block;
    const int64_t th = (t_total + tbs - 1) / tbs;
    const int64_t n_start = (int64_t)ep_rank * nr;
    memset(a, 0, sizeof(*a));
    a->t_total = t_total;
    a->th = th;
    a->nr = nr;
    a->partial_token_counts = zalloc64(nr * th);
    a->expert_counts = zalloc64(t_total);
    for (int64_t tid = 0; tid < th; ++tid)
        for (int64_t i = 0; i < tbs; ++i) {
            const int64_t t = tid * tbs + i;
            if (t >= t_total) break;
            for (int64_t k = 0; k < K; ++k) {
                const int64_t n = indices[t * K + k];
                if (!(n >= 0 && n < c->n_experts)) {
                    strcpy(g_err, "count_tokens: expert id out of range");
                    orc_artifacts_free(a);
                    return 1;
                }
                if (n >= n_start && n < n_start + nr) {
                    a->partial_token_counts[(n - n_start) * th + tid]++;
                    a->expert_counts[t]++;
                }
            }
        }
    /* prefix_sum (kernels.hpp:300-310): exclusive with the total appended */
    a->partial_cum = zalloc64(nr * th + 1);
    int64_t acc = 0;
    for (int64_t i = 0; i < nr * th; ++i) {
        a->partial_cum[i] = acc;
        acc += a->partial_token_counts[i];
    }
    a->partial_cum[nr * th] = acc;
    a->cum_expert_counts = zalloc64(t_total + 1);
    acc = 0;
    for (int64_t t = 0; t < t_total; ++t) {
        a->cum_expert_counts[t] = acc;
        acc += a->expert_counts[t];
    }
    a->cum_expert_counts[t_total] = acc;
    a->cum_token_counts = zalloc64(nr + 1);
    for (int64_t ln = 0; ln <= nr; ++ln) a->cum_token_counts[ln] = a->partial_cum[ln * th];
    a->token_counts = zalloc64(nr);
    for (int64_t ln = 0; ln < nr; ++ln)
        a->token_counts[ln] = a->cum_token_counts[ln + 1] - a->cum_token_counts[ln];
    a->rt = a->cum_token_counts[nr];

    /* generate_indices */
    const int64_t rt = a->rt;
    a->input_indices = zalloc64(rt);
    a->output_indices = zalloc64(rt);
    a->selected_k = zalloc64(rt);
    a->counter = zalloc64(nr * th);
    for (int64_t ln = 0; ln < nr; ++ln)
        for (int64_t tid = 0; tid < th; ++tid) a->counter[ln * th + tid] = a->partial_cum[ln * th + tid];
    int64_t* seen = zalloc64(t_total);
    for (int64_t tid = 0; tid < th; ++tid)
        for (int64_t i = 0; i < tbs; ++i) {
            const int64_t t = tid * tbs + i;
            if (t >= t_total) break;
            for (int64_t k = 0; k < K; ++k) {
                const int64_t n = indices[t * K + k];
                if (n < n_start || n >= n_start + nr) continue;
                const int64_t ln = n - n_start;
                const int64_t row = a->counter[ln * th + tid]++;
                const int64_t pos = a->cum_expert_counts[t] + seen[t];
                a->input_indices[row] = t;
                a->output_indices[pos] = row;
                a->selected_k[pos] = k;
                seen[t]++;
            }
        }
    free(seen);
    return 0;
}

/* same contract as ref_routing_artifacts (oracle/ref_shim.cpp) */
int orc_routing_artifacts(const orc_moe_cfg* c, int64_t t_total, const int64_t* indices, int ep_rank,
                          int64_t* out_sizes, int64_t* token_counts, int64_t* partial_token_counts,
                          int64_t* partial_cum, int64_t* cum_token_counts, int64_t* expert_counts,
                          int64_t* cum_expert_counts, int64_t* input_indices, int64_t* output_indices,
                          int64_t* selected_k, int64_t* counter) {
    orc_artifacts a;
    if (orc_artifacts_build(c, t_total, indices, ep_rank, &a)) return 1;
    const int64_t nr = a.nr, th = a.th, rt = a.rt;
    out_sizes[0] = th;
    out_sizes[1] = rt;
#define CP(dst, src, n) \
    if (dst && (n) > 0) memcpy(dst, src, 8 * (size_t)(n))
    CP(token_counts, a.token_counts, nr);
    CP(partial_token_counts, a.partial_token_counts, nr * th);
    CP(partial_cum, a.partial_cum, nr * th + 1);
    CP(cum_token_counts, a.cum_token_counts, nr + 1);
    CP(expert_counts, a.expert_counts, t_total);
    CP(cum_expert_counts, a.cum_expert_counts, t_total + 1);
    CP(input_indices, a.input_indices, rt);
    CP(output_indices, a.output_indices, rt);
    CP(selected_k, a.selected_k, rt);
    CP(counter, a.counter, nr * th);
#undef CP
    orc_artifacts_free(&a);
    return 0;
}

/* ---- templated MoE body, instantiated for f32 and f64 ------------------------------- */

#define T float
#define SFX(name) name##_f32
#include "moe_oracle_impl.h"
#undef T
#undef SFX
#define T double
#define SFX(name) name##_f64
#include "moe_oracle_impl.h"
#undef T
#undef SFX

int orc_route_f32(const orc_moe_cfg* c, int64_t s, const float* x, const float* router, float* logits,
                  float* probs, float* weights, int64_t* indices) {
    if (orc_validate(c)) return 1;
    return route_f32(c, s, x, router, logits, probs, weights, indices);
}

int orc_softmax_topk_f32(int64_t rows, int64_t n, int64_t k, const float* logits, float* probs,
                         float* values, int64_t* indices) {
    double* e = (double*)malloc(sizeof(double) * (size_t)n);
    char* taken = (char*)malloc((size_t)n);
    softmax_f32(logits, probs, rows, n, e);
    topk_f32(probs, rows, n, k, values, indices, taken);
    free(e);
    free(taken);
    return 0;
}

int orc_moe_layer_f32(const orc_moe_cfg* c, int64_t s, const float* x, const float* router,
                      const float* gate, const float* up, const float* down, const float* dout, int fur,
                      double aux_coeff, int do_backward, float* out, float* dx, float* drouter,
                      float* dgate, float* dup, float* ddown, float* weights, int64_t* idx, float* probs,
                      double* aux) {
    return moe_layer_f32(c, s, x, router, gate, up, down, dout, fur, aux_coeff, do_backward, out, dx,
                         drouter, dgate, dup, ddown, weights, idx, probs, aux);
}

int orc_moe_layer_f64(const orc_moe_cfg* c, int64_t s, const double* x, const double* router,
                      const double* gate, const double* up, const double* down, const double* dout,
                      int fur, double aux_coeff, int do_backward, double* out, double* dx, double* drouter,
                      double* dgate, double* dup, double* ddown, double* weights, int64_t* idx,
                      double* probs, double* aux) {
    return moe_layer_f64(c, s, x, router, gate, up, down, dout, fur, aux_coeff, do_backward, out, dx,
                         drouter, dgate, dup, ddown, weights, idx, probs, aux);
}

/* moe.hpp:471-497 reference_moe_forward (dense per-token oracle), full expert set [N,...] */
int orc_dense_moe_forward_f32(const orc_moe_cfg* c, int64_t t_total, const float* x, const float* gate,
                              const float* up, const float* down, const float* weights,
                              const int64_t* indices, float* out) {
    if (orc_validate(c)) return 1;
    if (dense_forward_f32(c, t_total, x, gate, up, down, weights, indices, out)) {
        strcpy(g_err, "reference_moe: expert id out of range");
        return 1;
    }
    return 0;
}

/* ---- optimizer (optim.cpp) ------------------------------------------------------------- */

typedef struct {
    double beta1, beta2, eps, weight_decay, peak_lr, min_lr;
    int64_t warmup_steps, total_steps;
    double clip_norm;
    int32_t clip_after_warmup_only, round_weights_bf16;
} orc_adamw_cfg;

void orc_adamw_default_cfg(orc_adamw_cfg* c) {
    c->beta1 = 0.9;
    c->beta2 = 0.99;
    c->eps = 1e-8;
    c->weight_decay = 0.1;
    c->peak_lr = 4e-4;
    c->min_lr = 4e-5;
    c->warmup_steps = 2500;
    c->total_steps = 100000;
    c->clip_norm = 1.0;
    c->clip_after_warmup_only = 1;
    c->round_weights_bf16 = 1;
}

/* optim.cpp:17-24 */
double orc_lr_at_step(int64_t step, const orc_adamw_cfg* c) {
    if (step < c->warmup_steps) return c->peak_lr * (double)step / (double)c->warmup_steps;
    if (step >= c->total_steps) return c->min_lr;
    const double t = (double)(step - c->warmup_steps) / (double)(c->total_steps - c->warmup_steps);
    return c->min_lr + 0.5 * (c->peak_lr - c->min_lr) * (1.0 + cos(M_PI * t));
}

/* optim.cpp:43-50: equal shares, remainder on the last member */
/* optim.cpp:196-221 memory_report; out = {weights, grads, master, optim, total, capacity, feasible} */
int orc_memory_report(int64_t p_expert, int64_t p_non_expert, int mode, int dp, int ep, double capacity_gb,
                      double* out) {
    if (p_expert < 0 || p_non_expert < 0) {
        strcpy(g_err, "memory_report: negative parameter count");
        return 1;
    }
    if (dp < 1 || ep < 1) {
        strcpy(g_err, "memory_report: bad group sizes");
        return 1;
    }
    const double p = (double)(p_expert + p_non_expert);
    double se = 1.0, sn = 1.0;
    if (mode == 1) se = sn = 1.0 / dp;
    if (mode == 2) {
        se = 1.0 / dp;
        sn = 1.0 / ((double)dp * ep);
    }
    out[0] = 2.0 * p;
    out[1] = 2.0 * p;
    out[2] = 4.0 * ((double)p_expert * se + (double)p_non_expert * sn);
    out[3] = 2.0 * out[2];
    out[4] = out[0] + out[1] + out[2] + out[3];
    out[5] = capacity_gb * 1e9;
    out[6] = out[4] <= out[5] ? 1.0 : 0.0;
    return 0;
}

int orc_shard_slice(int64_t numel, int g, int pos, int64_t* begin, int64_t* end) {
    if (!(g >= 1 && pos >= 0 && pos < g)) {
        strcpy(g_err, "shard_slice: bad position");
        return 1;
    }
    const int64_t base = numel / g;
    *begin = (int64_t)pos * base;
    *end = pos == g - 1 ? numel : *begin + base;
    return 0;
}

/* optim.cpp:88-107: decay on the master, fp64 moments rounded to fp32, bias-corrected step */
int orc_adamw_update(float* master, float* m, float* v, const float* grad, int64_t n, double lr,
                     int64_t step, const orc_adamw_cfg* c, float* weight_out, int round_bf16) {
    const double bc1 = 1.0 - pow(c->beta1, (double)(step + 1));
    const double bc2 = 1.0 - pow(c->beta2, (double)(step + 1));
    for (int64_t i = 0; i < n; ++i) {
        double w = master[i];
        const double g = grad[i];
        w -= lr * c->weight_decay * w;
        const double mm = c->beta1 * m[i] + (1.0 - c->beta1) * g;
        const double vv = c->beta2 * v[i] + (1.0 - c->beta2) * g * g;
        m[i] = (float)mm;
        v[i] = (float)vv;
        w -= lr * ((double)m[i] / bc1) / (sqrt((double)v[i] / bc2) + c->eps);
        master[i] = (float)w;
        weight_out[i] = round_bf16 ? orc_bf16_round(master[i]) : master[i];
    }
    return 0;
}

/* rank layout comm.hpp:45-59 with pp = 0: rank = (dp*EP + ep)*TP + tp */
static int rank_of3(int dp, int ep, int tp, int EP, int TP) { return (dp * EP + ep) * TP + tp; }

/* optim.cpp:74-86 */
static int counts_toward_norm(int mode, int cls, int tp_sharded, int dp, int ep, int tp) {
    if (!tp_sharded && tp != 0) return 0;
    if (mode == 0) return dp == 0 && (cls == 1 || ep == 0);
    if (mode == 1) return cls == 1 || ep == 0;
    return 1;
}

/* ShardedOptimizer over a simulated dp x ep x tp world; same contract as
 * ref_sharded_steps in ref_shim.cpp (mode: 0 ddp, 1 so, 2 epso). */
int orc_sharded_steps(int DP, int EP, int TP, int mode, const orc_adamw_cfg* c, int nparams,
                      const int64_t* numel, const int* cls, const int* tp_sharded, const float* w_init,
                      const float* grads, int steps, float* w_out, float* master_out, float* m_out,
                      float* v_out, int64_t* owned_out, double* stats_out, int64_t* state_bytes_out) {
    const int W = DP * EP * TP;
    int64_t total = 0, maxn = 0;
    int64_t* off = (int64_t*)calloc((size_t)nparams + 1, 8);
    for (int p = 0; p < nparams; ++p) {
        off[p] = total;
        total += numel[p];
        if (numel[p] > maxn) maxn = numel[p];
    }
    off[nparams] = total;
    /* plan: owned slice per rank per param (optim.cpp:52-72) */
    int64_t* own_b = (int64_t*)calloc((size_t)(W * nparams), 8);
    int64_t* own_e = (int64_t*)calloc((size_t)(W * nparams), 8);
    for (int r = 0; r < W; ++r) {
        const int tp = r % TP, ep = (r / TP) % EP, dp = r / (TP * EP);
        for (int p = 0; p < nparams; ++p) {
            if (mode == 0) {
                own_b[r * nparams + p] = 0;
                own_e[r * nparams + p] = numel[p];
            } else {
                const int over = mode == 2 && cls[p] == 0;
                const int g = over ? DP * EP : DP;
                const int pos = over ? dp * EP + ep : dp;
                orc_shard_slice(numel[p], g, pos, &own_b[r * nparams + p], &own_e[r * nparams + p]);
            }
        }
    }
    (void)tp_sharded;
    float* w = (float*)malloc(sizeof(float) * (size_t)(W * total));
    memcpy(w, w_init, sizeof(float) * (size_t)(W * total));
    /* states: per rank, owned slices packed in param order at the param's offset */
    float* master = (float*)calloc((size_t)(W * total), 4);
    float* mm = (float*)calloc((size_t)(W * total), 4);
    float* vv = (float*)calloc((size_t)(W * total), 4);
    for (int r = 0; r < W; ++r)
        for (int p = 0; p < nparams; ++p) {
            const int64_t b = own_b[r * nparams + p], e = own_e[r * nparams + p];
            memcpy(master + r * total + off[p], w + r * total + off[p] + b, 4 * (size_t)(e - b));
        }
    float* synced = (float*)calloc((size_t)(W * total), 4);  /* per rank, owned slice of each param */
    float* tmp = (float*)calloc((size_t)(maxn + 1), 4);
    float* tmp2 = (float*)calloc((size_t)(maxn + 1), 4);
    float* upd = (float*)calloc((size_t)(W * total), 4);
    int64_t step_count = 0;
    for (int s = 0; s < steps; ++s) {
        const float* G = grads + (int64_t)s * W * total;
        const double lr = orc_lr_at_step(step_count, c);
        /* 1. gradient sync per rank */
        for (int r = 0; r < W; ++r) {
            const int tp = r % TP, ep = (r / TP) % EP, dp = r / (TP * EP);
            for (int p = 0; p < nparams; ++p) {
                const int64_t n = numel[p];
                /* per-member flat grads after the optional SO pre-average over EP */
#define FLAT_OF(dst, rr)                                                                           \
    do {                                                                                           \
        const int tp_ = (rr) % TP, ep_ = ((rr) / TP) % EP, dp_ = (rr) / (TP * EP);                 \
        (void)ep_;                                                                                 \
        if (cls[p] == 0 && mode != 2 && EP > 1) {                                                  \
            for (int64_t i = 0; i < n; ++i) dst[i] = G[(int64_t)rank_of3(dp_, 0, tp_, EP, TP) * total + off[p] + i]; \
            for (int e2 = 1; e2 < EP; ++e2)                                                        \
                for (int64_t i = 0; i < n; ++i)                                                    \
                    dst[i] += G[(int64_t)rank_of3(dp_, e2, tp_, EP, TP) * total + off[p] + i];     \
            const float sc = (float)(1.0 / (double)EP);                                            \
            for (int64_t i = 0; i < n; ++i) dst[i] *= sc;                                          \
        } else {                                                                                   \
            for (int64_t i = 0; i < n; ++i) dst[i] = G[(int64_t)(rr) * total + off[p] + i];       \
        }                                                                                          \
    } while (0)
                if (mode == 0) {
                    /* allreduce_mean over DP (members in dp order) */
                    FLAT_OF(tmp, rank_of3(0, ep, tp, EP, TP));
                    for (int d = 1; d < DP; ++d) {
                        FLAT_OF(tmp2, rank_of3(d, ep, tp, EP, TP));
                        for (int64_t i = 0; i < n; ++i) tmp[i] += tmp2[i];
                    }
                    const float sc = (float)(1.0 / (double)DP);
                    for (int64_t i = 0; i < n; ++i) synced[r * total + off[p] + i] = tmp[i] * sc;
                } else {
                    const int over = mode == 2 && cls[p] == 0;
                    const int g = over ? DP * EP : DP;
                    const int64_t b = own_b[r * nparams + p], e = own_e[r * nparams + p];
                    for (int m2 = 0; m2 < g; ++m2) {
                        const int rr = over ? rank_of3(m2 / EP, m2 % EP, tp, EP, TP) : rank_of3(m2, ep, tp, EP, TP);
                        FLAT_OF(tmp2, rr);
                        for (int64_t i = b; i < e; ++i) {
                            if (m2 == 0) tmp[i] = tmp2[i];
                            else tmp[i] += tmp2[i];
                        }
                    }
                    const float sc = (float)(1.0 / (double)g);
                    for (int64_t i = b; i < e; ++i) synced[r * total + off[p] + (i - b)] = tmp[i] * sc;
                }
#undef FLAT_OF
                (void)dp;
            }
        }
        /* 2. global norm: per-rank fp64 partials, world allreduce in rank order */
        double world_sq = 0;
        for (int r = 0; r < W; ++r) {
            const int tp = r % TP, ep = (r / TP) % EP, dp = r / (TP * EP);
            double partial = 0;
            for (int p = 0; p < nparams; ++p)
                if (counts_toward_norm(mode, cls[p], tp_sharded[p], dp, ep, tp)) {
                    const int64_t len = own_e[r * nparams + p] - own_b[r * nparams + p];
                    for (int64_t i = 0; i < len; ++i) {
                        const float gv = synced[r * total + off[p] + i];
                        partial += (double)gv * (double)gv;
                    }
                }
            if (r == 0) world_sq = partial;
            else world_sq += partial;
        }
        const double norm = sqrt(world_sq);
        double clip = 1.0;
        const int active = !c->clip_after_warmup_only || step_count >= c->warmup_steps;
        if (active && norm > c->clip_norm && norm > 0) clip = c->clip_norm / norm;
        /* 3-4. update owned slices */
        for (int r = 0; r < W; ++r) {
            for (int p = 0; p < nparams; ++p) {
                const int64_t len = own_e[r * nparams + p] - own_b[r * nparams + p];
                float* gs = synced + r * total + off[p];
                if (clip != 1.0)
                    for (int64_t i = 0; i < len; ++i) gs[i] = (float)((double)gs[i] * clip);
                orc_adamw_update(master + r * total + off[p], mm + r * total + off[p], vv + r * total + off[p],
                                 gs, len, lr, step_count, c, upd + r * total + off[p], c->round_weights_bf16);
            }
            double* so = stats_out + ((int64_t)s * W + r) * 3;
            so[0] = lr;
            so[1] = norm;
            so[2] = clip;
        }
        /* re-share: allgatherv over the owning group (member order) */
        for (int r = 0; r < W; ++r) {
            const int tp = r % TP, ep = (r / TP) % EP;
            for (int p = 0; p < nparams; ++p) {
                if (mode == 0) {
                    memcpy(w + r * total + off[p], upd + r * total + off[p], 4 * (size_t)numel[p]);
                    continue;
                }
                const int over = mode == 2 && cls[p] == 0;
                const int g = over ? DP * EP : DP;
                for (int m2 = 0; m2 < g; ++m2) {
                    const int rr = over ? rank_of3(m2 / EP, m2 % EP, tp, EP, TP) : rank_of3(m2, ep, tp, EP, TP);
                    const int64_t b = own_b[rr * nparams + p], e = own_e[rr * nparams + p];
                    memcpy(w + r * total + off[p] + b, upd + rr * total + off[p], 4 * (size_t)(e - b));
                }
            }
        }
        step_count++;
    }
    memcpy(w_out, w, sizeof(float) * (size_t)(W * total));
    for (int r = 0; r < W; ++r) {
        int64_t packed = 0, owned = 0;
        for (int p = 0; p < nparams; ++p) {
            const int64_t b = own_b[r * nparams + p], e = own_e[r * nparams + p];
            owned_out[((int64_t)r * nparams + p) * 2 + 0] = b;
            owned_out[((int64_t)r * nparams + p) * 2 + 1] = e;
            memcpy(master_out + r * total + packed, master + r * total + off[p], 4 * (size_t)(e - b));
            memcpy(m_out + r * total + packed, mm + r * total + off[p], 4 * (size_t)(e - b));
            memcpy(v_out + r * total + packed, vv + r * total + off[p], 4 * (size_t)(e - b));
            packed += e - b;
            owned += e - b;
        }
        state_bytes_out[r] = 12 * owned;
    }
    free(off);
    free(own_b);
    free(own_e);
    free(w);
    free(master);
    free(mm);
    free(vv);
    free(synced);
    free(tmp);
    free(tmp2);
    free(upd);
    return 0;
}

/* ---- record files (reliability.hpp:33-70, reliability.cpp:23-320) -------------------------
 * Layout: "OPTT", u32 version 1, u32 count, per record {u32 name length, name, u32 dtype
 * (0 f32, 1 bf16), u32 ndim, u64 dims, payload LE}, then u32 zlib crc32 of all of it.
 * Records are given as NUL-separated names plus f32 data, all records concatenated;
 * bf16 records round with orc_f32_to_bf16_bits (RecordFileWriter::add_bf16, 238-253). */

uint32_t orc_crc32(uint32_t crc, const uint8_t* p, int64_t n) { /* zlib crc32, bitwise */
    uint32_t r = ~crc;
    for (int64_t i = 0; i < n; ++i) {
        r ^= p[i];
        for (int b = 0; b < 8; ++b) r = (r & 1u) ? (r >> 1) ^ 0xEDB88320u : r >> 1;
    }
    return ~r;
}

static void put_le(uint8_t* out, int64_t* at, uint64_t v, int bytes) {
    for (int i = 0; i < bytes; ++i) {
        if (out) out[*at] = (uint8_t)((v >> (8 * i)) & 0xff);
        ++*at;
    }
}
static uint64_t get_le(const uint8_t* b, int bytes) {
    uint64_t v = 0;
    for (int i = 0; i < bytes; ++i) v |= (uint64_t)b[i] << (8 * i);
    return v;
}

/* serialise into out (NULL: size query); returns the file size, or -1 on a bad record */
int64_t orc_record_file_bytes(int n_rec, const char* names, const int32_t* dtypes, const int32_t* ndims,
                              const int64_t* dims, const float* data, uint8_t* out) {
    int64_t at = 0, di = 0, de = 0;
    const char magic[4] = {'O', 'P', 'T', 'T'};
    for (int i = 0; i < 4; ++i) put_le(out, &at, (uint8_t)magic[i], 1);
    put_le(out, &at, 1, 4);
    put_le(out, &at, (uint64_t)n_rec, 4);
    for (int r = 0; r < n_rec; ++r) {
        const size_t len = strlen(names);
        put_le(out, &at, len, 4);
        for (size_t c = 0; c < len; ++c) put_le(out, &at, (uint8_t)names[c], 1);
        names += len + 1;
        if (dtypes[r] < 0 || dtypes[r] > 1 || ndims[r] < 0 || ndims[r] > 8) {
            strcpy(g_err, "record: bad dtype or rank");
            return -1;
        }
        put_le(out, &at, (uint64_t)dtypes[r], 4);
        put_le(out, &at, (uint64_t)ndims[r], 4);
        int64_t n = 1;
        for (int d = 0; d < ndims[r]; ++d) {
            if (dims[di] < 0) {
                strcpy(g_err, "record: negative dimension");
                return -1;
            }
            n *= dims[di];
            put_le(out, &at, (uint64_t)dims[di++], 8);
        }
        for (int64_t e = 0; e < n; ++e, ++de) {
            if (dtypes[r] == 0) {
                uint32_t u;
                memcpy(&u, &data[de], 4);
                put_le(out, &at, u, 4);
            } else {
                put_le(out, &at, orc_f32_to_bf16_bits(data[de]), 2);
            }
        }
    }
    const int64_t body = at;
    put_le(out, &at, out ? orc_crc32(0, out, body) : 0, 4);
    return at;
}

/* read_record_file: 0 and the record count / total elements (data_out: the records
 * widened to f32 and concatenated, cap elements) or 1 with the reference's message */
int orc_record_file_parse(const uint8_t* b, int64_t size, int64_t* count, int64_t* total, float* data_out,
                          int64_t cap) {
#define BAD(msg)                \
    do {                        \
        strcpy(g_err, msg);     \
        return 1;               \
    } while (0)
    if (size < 16) BAD("truncated header");
    if (memcmp(b, "OPTT", 4) != 0) BAD("bad magic");
    if (get_le(b + 4, 4) != 1) BAD("unsupported version");
    if (orc_crc32(0, b, size - 4) != (uint32_t)get_le(b + size - 4, 4)) BAD("checksum mismatch");
    const uint32_t cnt = (uint32_t)get_le(b + 8, 4);
    const int64_t end = size - 4;
    int64_t off = 12, tot = 0;
    for (uint32_t r = 0; r < cnt; ++r) {
        if (end - off < 4) BAD("truncated record");
        const uint32_t name_len = (uint32_t)get_le(b + off, 4);
        off += 4;
        if (name_len > 4096) BAD("oversized record name");
        if (end - off < name_len) BAD("truncated record");
        off += name_len;
        if (end - off < 8) BAD("truncated record");
        const uint32_t dt = (uint32_t)get_le(b + off, 4), nd = (uint32_t)get_le(b + off + 4, 4);
        off += 8;
        if (dt > 1) BAD("unknown dtype");
        if (nd > 8) BAD("too many dimensions");
        if (end - off < (int64_t)nd * 8) BAD("truncated record");
        int64_t n = 1;
        for (uint32_t d = 0; d < nd; ++d, off += 8) n *= (int64_t)get_le(b + off, 8);
        const int64_t payload = n * (dt == 0 ? 4 : 2);
        if (end - off < payload) BAD("truncated record");
        for (int64_t e = 0; e < n && data_out; ++e) {
            if (tot + e >= cap) break;
            uint32_t u = dt == 0 ? (uint32_t)get_le(b + off + 4 * e, 4) : (uint32_t)get_le(b + off + 2 * e, 2) << 16;
            memcpy(&data_out[tot + e], &u, 4);
        }
        off += payload;
        tot += n;
    }
    if (off != end) BAD("trailing bytes after last record");
#undef BAD
    *count = cnt;
    *total = tot;
    return 0;
}
