/* TEST INFRASTRUCTURE ONLY — the CPU restatement of the reference's MoE
 * algorithm (FastSparseMoE, Algorithm 1) used as the parity checker.
 * Instantiated twice by moe_oracle.c with T = float / double (the reference's
 * templates are <T>: include/optimus/moe.hpp:344-466).
 *
 * Loop orders follow the reference line by line so that, compiled with
 * -ffp-contract=off (what g++ -std=c++20 does for the reference), results are
 * bitwise identical to it; tests/test_oracle_pin.py checks exactly that against
 * oracle/_ref (the reference compiled in place).
 *
 * Required macros: T (element type), SFX(name) (name suffixing). */

/* kernels.hpp:16-49 matmul, non-f64 path: out[i,j] += a[i,p] * b[p,j], p outer */
static void SFX(matmul)(const T* a, const T* b, T* out, int64_t m, int64_t k, int64_t n) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < m; ++i) {
        T* op = out + i * n;
        for (int64_t j = 0; j < n; ++j) op[j] = (T)0;
        for (int64_t p = 0; p < k; ++p) {
            const T av = a[i * k + p];
            const T* bp = b + p * n;
            for (int64_t j = 0; j < n; ++j) op[j] += av * bp[j];
        }
    }
}

/* kernels.hpp:52-72 matmul_tn: a [K,M], b [K,N] -> [M,N] (accumulates into zeroed out) */
static void SFX(matmul_tn)(const T* a, const T* b, T* out, int64_t k, int64_t m, int64_t n) {
    /* the reference runs p outer, i inner; every out[i,j] still accumulates p = 0..k-1 in
     * order here (i outer, split across threads), so the result is bitwise the same */
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < m; ++i) {
        T* op = out + i * n;
        for (int64_t j = 0; j < n; ++j) op[j] = (T)0;
        for (int64_t p = 0; p < k; ++p) {
            const T av = a[p * m + i];
            const T* bp = b + p * n;
            for (int64_t j = 0; j < n; ++j) op[j] += av * bp[j];
        }
    }
}

/* kernels.hpp:75-96 matmul_nt: a [M,K], b [N,K] -> [M,N] */
static void SFX(matmul_nt)(const T* a, const T* b, T* out, int64_t m, int64_t k, int64_t n) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < m; ++i) {
        const T* ap = a + i * k;
        T* op = out + i * n;
        for (int64_t j = 0; j < n; ++j) {
            const T* bp = b + j * k;
            T acc = 0;
            for (int64_t p = 0; p < k; ++p) acc += ap[p] * bp[p];
            op[j] = acc;
        }
    }
}

/* kernels.hpp:111-134 grouped_mm: rows [b[g], b[g+1]) x weights[g] ([G,K1,K2]) */
static void SFX(grouped_mm)(const T* in, const T* w, const int64_t* bnd, int64_t groups,
                            int64_t rows, int64_t k1, int64_t k2, T* out) {
    for (int64_t i = 0; i < rows * k2; ++i) out[i] = (T)0;
    for (int64_t g = 0; g < groups; ++g) {
        const T* wg = w + g * k1 * k2;
#pragma omp parallel for schedule(static)
        for (int64_t i = bnd[g]; i < bnd[g + 1]; ++i) {
            T* op = out + i * k2;
            const T* ip = in + i * k1;
            for (int64_t p = 0; p < k1; ++p) {
                const T av = ip[p];
                const T* wp = wg + p * k2;
                for (int64_t j = 0; j < k2; ++j) op[j] += av * wp[j];
            }
        }
    }
}

/* kernels.hpp:137-162 grouped_mm_nt: input [R,K2] x weights[g]^T -> [R,K1] */
static void SFX(grouped_mm_nt)(const T* in, const T* w, const int64_t* bnd, int64_t groups,
                               int64_t rows, int64_t k1, int64_t k2, T* out) {
    for (int64_t i = 0; i < rows * k1; ++i) out[i] = (T)0;
    for (int64_t g = 0; g < groups; ++g) {
        const T* wg = w + g * k1 * k2;
#pragma omp parallel for schedule(static)
        for (int64_t i = bnd[g]; i < bnd[g + 1]; ++i) {
            const T* ip = in + i * k2;
            T* op = out + i * k1;
            for (int64_t p = 0; p < k1; ++p) {
                const T* wp = wg + p * k2;
                T acc = 0;
                for (int64_t j = 0; j < k2; ++j) acc += ip[j] * wp[j];
                op[p] = acc;
            }
        }
    }
}

/* kernels.hpp:165-189 grouped_mm_weight_grad: x [R,K1], dy [R,K2] -> [G,K1,K2] */
static void SFX(grouped_wgrad)(const T* x, const T* dy, const int64_t* bnd, int64_t groups,
                               int64_t k1, int64_t k2, T* out) {
    /* the reference runs rows i outer, p inner; every out[g,p,j] still accumulates its
     * group's rows in ascending order here (p rows split across threads) -> bitwise equal */
    for (int64_t i = 0; i < groups * k1 * k2; ++i) out[i] = (T)0;
    for (int64_t g = 0; g < groups; ++g) {
        T* wg = out + g * k1 * k2;
#pragma omp parallel for schedule(static)
        for (int64_t p = 0; p < k1; ++p) {
            T* wp = wg + p * k2;
            for (int64_t i = bnd[g]; i < bnd[g + 1]; ++i) {
                const T xv = x[i * k1 + p];
                const T* dp = dy + i * k2;
                for (int64_t j = 0; j < k2; ++j) wp[j] += xv * dp[j];
            }
        }
    }
}

/* kernels.hpp:194-214 softmax: max in T, exp/sum in double, cast */
static void SFX(softmax)(const T* x, T* out, int64_t rows, int64_t n, double* e) {
    for (int64_t i = 0; i < rows; ++i) {
        const T* xp = x + i * n;
        T mx = xp[0];
        for (int64_t j = 1; j < n; ++j) mx = (mx < xp[j]) ? xp[j] : mx; /* std::max(a,b) = a<b?b:a */
        double sum = 0.0;
        for (int64_t j = 0; j < n; ++j) {
            e[j] = exp((double)xp[j] - (double)mx);
            sum += e[j];
        }
        T* op = out + i * n;
        for (int64_t j = 0; j < n; ++j) op[j] = (T)(e[j] / sum);
    }
}

/* kernels.hpp:217-232 softmax_backward */
static void SFX(softmax_backward)(const T* probs, const T* dprobs, T* out, int64_t rows, int64_t n) {
    for (int64_t i = 0; i < rows; ++i) {
        const T* pp = probs + i * n;
        const T* dp = dprobs + i * n;
        double dot = 0.0;
        for (int64_t j = 0; j < n; ++j) dot += (double)pp[j] * (double)dp[j];
        T* op = out + i * n;
        for (int64_t j = 0; j < n; ++j) op[j] = (T)((double)pp[j] * ((double)dp[j] - dot));
    }
}

/* kernels.hpp:235-258 topk: K argmax rounds, strict '>' => ties to the lower index */
static void SFX(topk)(const T* probs, int64_t rows, int64_t n, int64_t k, T* values,
                      int64_t* indices, char* taken) {
    for (int64_t i = 0; i < rows; ++i) {
        const T* pp = probs + i * n;
        memset(taken, 0, (size_t)n);
        for (int64_t c = 0; c < k; ++c) {
            int64_t best = -1;
            for (int64_t j = 0; j < n; ++j) {
                if (taken[j]) continue;
                if (best < 0 || pp[j] > pp[best]) best = j;
            }
            taken[best] = 1;
            values[i * k + c] = pp[best];
            indices[i * k + c] = best;
        }
    }
}

/* moe.hpp:58-80 route (+ optional renormalisation, 72-78) */
static int SFX(route)(const orc_moe_cfg* c, int64_t s, const T* x, const T* router, T* logits,
                      T* probs, T* weights, int64_t* indices) {
    const int64_t H = c->hidden, N = c->n_experts, K = c->top_k;
    SFX(matmul)(x, router, logits, s, H, N);
    double* e = (double*)malloc(sizeof(double) * (size_t)N);
    char* taken = (char*)malloc((size_t)N);
    SFX(softmax)(logits, probs, s, N, e);
    SFX(topk)(probs, s, N, K, weights, indices, taken);
    free(e);
    free(taken);
    if (c->normalize_topk) {
        for (int64_t r = 0; r < s; ++r) {
            T sum = 0;
            for (int64_t k = 0; k < K; ++k) sum += weights[r * K + k];
            for (int64_t k = 0; k < K; ++k) weights[r * K + k] /= sum;
        }
    }
    return 0;
}

static double SFX(silu_scalar)(double x) { return x / (1.0 + exp(-x)); }

/* One MoE layer forward (+ backward) with the EP world simulated in-process:
 * allgather = rank-order concatenation (comm.hpp:326-347), reducescatter =
 * rank-order sum then chunk (comm.hpp:377-414). Same argument contract as
 * ref_moe_layer_* in ref_shim.cpp. */
static int SFX(moe_layer)(const orc_moe_cfg* c, int64_t S, const T* x_full, const T* router,
                          const T* gate_full, const T* up_full, const T* down_full,
                          const T* dout_full, int fur, double aux_coeff, int do_backward,
                          T* out_full, T* dx_full, T* drouter, T* dgate, T* dup, T* ddown,
                          T* weights_out, int64_t* idx_out, T* probs_out, double* aux_out) {
    if (orc_validate(c)) return 1;
    const int EP = c->ep;
    const int64_t H = c->hidden, I = c->intermediate, N = c->n_experts, K = c->top_k;
    const int64_t NR = N / EP, T_tot = (int64_t)EP * S, blk = H * I;

    /* stage 1: local routing per rank, then the gathered tables */
    T* logits = (T*)calloc((size_t)(T_tot * N), sizeof(T));
    T* probs = (T*)calloc((size_t)(T_tot * N), sizeof(T));
    T* w_g = (T*)calloc((size_t)(T_tot * K), sizeof(T));       /* gathered weights */
    int64_t* i_g = (int64_t*)calloc((size_t)(T_tot * K), 8);    /* gathered indices */
    T* r_w = (T*)calloc((size_t)(T_tot * K), sizeof(T));       /* routing.weights (learned) */
    int64_t* r_i = (int64_t*)calloc((size_t)(T_tot * K), 8);
    for (int r = 0; r < EP; ++r) {
        SFX(route)(c, S, x_full + r * S * H, router, logits + r * S * N, probs + r * S * N,
                   r_w + r * S * K, r_i + r * S * K);
    }
    for (int64_t t = 0; t < T_tot; ++t)
        for (int64_t k = 0; k < K; ++k) {
            if (fur) {
                const int64_t tl = t % S; /* fur_route is per rank over its S tokens */
                w_g[t * K + k] = (T)(1.0 / (double)K);
                i_g[t * K + k] = (tl * K + k) % N;
            } else {
                w_g[t * K + k] = r_w[t * K + k];
                i_g[t * K + k] = r_i[t * K + k];
            }
        }
    if (weights_out) memcpy(weights_out, r_w, sizeof(T) * (size_t)(T_tot * K));
    if (idx_out) memcpy(idx_out, r_i, 8 * (size_t)(T_tot * K));
    if (probs_out) memcpy(probs_out, probs, sizeof(T) * (size_t)(T_tot * N));

    /* balancing statistics (moe.hpp:381-386): sel over the gathered table, mean over local rows */
    int64_t* sel = (int64_t*)calloc((size_t)N, 8);
    for (int64_t i = 0; i < T_tot * K; ++i) sel[i_g[i]]++;
    T* mean_probs = (T*)calloc((size_t)(EP * N), sizeof(T));
    for (int r = 0; r < EP; ++r) {
        T* mp = mean_probs + r * N;
        for (int64_t row = 0; row < S; ++row)
            for (int64_t e = 0; e < N; ++e) mp[e] += probs[(r * S + row) * N + e];
        const T sc = (T)(1.0 / (double)S);
        for (int64_t e = 0; e < N; ++e) mp[e] *= sc;
        if (aux_out) {
            const double total = (double)T_tot * (double)K;
            double acc = 0;
            for (int64_t e = 0; e < N; ++e) acc += ((double)sel[e] / total) * (double)mp[e];
            aux_out[r] = (double)N * acc;
        }
    }

    /* per-rank expert work on the gathered rows */
    T* combined = (T*)calloc((size_t)(EP * T_tot * H), sizeof(T)); /* [EP][T,H] partials */
    T* wgrad_full = (T*)calloc((size_t)(EP * T_tot * K), sizeof(T));
    T* dgathered = (T*)calloc((size_t)(EP * T_tot * H), sizeof(T));
    orc_artifacts* arts = (orc_artifacts*)calloc((size_t)EP, sizeof(orc_artifacts));
    T** cache = (T**)calloc((size_t)EP * 5, sizeof(T*));
    for (int r = 0; r < EP; ++r) {
        orc_artifacts* a = &arts[r];
        if (orc_artifacts_build(c, T_tot, i_g, r, a)) return 1;
        const int64_t RT = a->rt;
        const T* wg = gate_full + (int64_t)r * NR * blk;
        const T* wu = up_full + (int64_t)r * NR * blk;
        const T* wd = down_full + (int64_t)r * NR * blk;
        T* mlp_in = (T*)calloc((size_t)(RT * H + 1), sizeof(T));
        T* g_out = (T*)calloc((size_t)(RT * I + 1), sizeof(T));
        T* u_out = (T*)calloc((size_t)(RT * I + 1), sizeof(T));
        T* mul = (T*)calloc((size_t)(RT * I + 1), sizeof(T));
        T* mlp_out = (T*)calloc((size_t)(RT * H + 1), sizeof(T));
        /* moe.hpp:225-244 expert_forward */
        for (int64_t row = 0; row < RT; ++row)
            memcpy(mlp_in + row * H, x_full + a->input_indices[row] * H, sizeof(T) * (size_t)H);
        SFX(grouped_mm)(mlp_in, wg, a->cum_token_counts, NR, RT, H, I, g_out);
        SFX(grouped_mm)(mlp_in, wu, a->cum_token_counts, NR, RT, H, I, u_out);
        for (int64_t i = 0; i < RT * I; ++i)
            mul[i] = (T)(SFX(silu_scalar)((double)g_out[i]) * (double)u_out[i]);
        SFX(grouped_mm)(mul, wd, a->cum_token_counts, NR, RT, I, H, mlp_out);
        /* moe.hpp:250-268 output_reduction_forward */
        T* comb = combined + (int64_t)r * T_tot * H;
        for (int64_t t = 0; t < T_tot; ++t) {
            T* op = comb + t * H;
            for (int64_t j = a->cum_expert_counts[t]; j < a->cum_expert_counts[t + 1]; ++j) {
                const int64_t row = a->output_indices[j];
                const T wv = w_g[t * K + a->selected_k[j]];
                const T* mp = mlp_out + row * H;
                for (int64_t cc = 0; cc < H; ++cc) op[cc] += wv * mp[cc];
            }
        }
        cache[r * 5 + 0] = mlp_in;
        cache[r * 5 + 1] = g_out;
        cache[r * 5 + 2] = u_out;
        cache[r * 5 + 3] = mul;
        cache[r * 5 + 4] = mlp_out;
    }
    /* reducescatter of the combined partials: rank-order sum, keep own chunk */
    for (int r = 0; r < EP; ++r)
        for (int64_t i = 0; i < S * H; ++i) {
            T acc = combined[(int64_t)0 * T_tot * H + r * S * H + i];
            for (int m = 1; m < EP; ++m) acc += combined[(int64_t)m * T_tot * H + r * S * H + i];
            out_full[r * S * H + i] = acc;
        }

    if (do_backward) {
        /* moe.hpp:392-466 fast_moe_backward; dout_full is already the allgather (400) */
        for (int r = 0; r < EP; ++r) {
            orc_artifacts* a = &arts[r];
            const int64_t RT = a->rt;
            const T* wg = gate_full + (int64_t)r * NR * blk;
            const T* wu = up_full + (int64_t)r * NR * blk;
            const T* wd = down_full + (int64_t)r * NR * blk;
            T *mlp_in = cache[r * 5 + 0], *g_out = cache[r * 5 + 1], *u_out = cache[r * 5 + 2];
            T *mul = cache[r * 5 + 3], *mlp_out = cache[r * 5 + 4];
            T* mog = (T*)calloc((size_t)(RT * H + 1), sizeof(T));
            T* wgr = wgrad_full + (int64_t)r * T_tot * K;
            /* moe.hpp:271-298 output_reduction_backward */
            for (int64_t t = 0; t < T_tot; ++t) {
                const T* gp = dout_full + t * H;
                for (int64_t j = a->cum_expert_counts[t]; j < a->cum_expert_counts[t + 1]; ++j) {
                    const int64_t row = a->output_indices[j];
                    const int64_t k = a->selected_k[j];
                    const T wv = w_g[t * K + k];
                    T* mg = mog + row * H;
                    const T* mp = mlp_out + row * H;
                    double dot = 0;
                    for (int64_t cc = 0; cc < H; ++cc) {
                        mg[cc] = wv * gp[cc];
                        dot += (double)gp[cc] * (double)mp[cc];
                    }
                    wgr[t * K + k] += (T)dot;
                }
            }
            T* dmul = (T*)calloc((size_t)(RT * I + 1), sizeof(T));
            SFX(grouped_mm_nt)(mog, wd, a->cum_token_counts, NR, RT, I, H, dmul);
            T* dd = ddown + (int64_t)r * NR * blk;
            SFX(grouped_wgrad)(mul, mog, a->cum_token_counts, NR, I, H, dd);
            T* dgo = (T*)calloc((size_t)(RT * I + 1), sizeof(T));
            T* duo = (T*)calloc((size_t)(RT * I + 1), sizeof(T));
            /* kernels.hpp:277-295 silu_glu_backward */
            for (int64_t i = 0; i < RT * I; ++i) {
                const double xv = (double)g_out[i];
                const double s = 1.0 / (1.0 + exp(-xv));
                const double dsilu = s * (1.0 + xv * (1.0 - s));
                duo[i] = (T)(SFX(silu_scalar)(xv) * (double)dmul[i]);
                dgo[i] = (T)((double)u_out[i] * (double)dmul[i] * dsilu);
            }
            T* dg = dgate + (int64_t)r * NR * blk;
            T* du = dup + (int64_t)r * NR * blk;
            SFX(grouped_wgrad)(mlp_in, dgo, a->cum_token_counts, NR, H, I, dg);
            SFX(grouped_wgrad)(mlp_in, duo, a->cum_token_counts, NR, H, I, du);
            T* dmi = (T*)calloc((size_t)(RT * H + 1), sizeof(T));
            T* dmi2 = (T*)calloc((size_t)(RT * H + 1), sizeof(T));
            SFX(grouped_mm_nt)(dgo, wg, a->cum_token_counts, NR, RT, H, I, dmi);
            SFX(grouped_mm_nt)(duo, wu, a->cum_token_counts, NR, RT, H, I, dmi2);
            for (int64_t i = 0; i < RT * H; ++i) dmi[i] += dmi2[i];
            T* dgath = dgathered + (int64_t)r * T_tot * H;
            for (int64_t row = 0; row < RT; ++row) {
                T* gp = dgath + a->input_indices[row] * H;
                const T* mp = dmi + row * H;
                for (int64_t cc = 0; cc < H; ++cc) gp[cc] += mp[cc];
            }
            /* moe.hpp:456-461: expert grads scaled to the mean-over-ranks objective */
            const T inv_ep = (T)(1.0 / (double)EP);
            for (int64_t i = 0; i < NR * blk; ++i) {
                dg[i] *= inv_ep;
                du[i] *= inv_ep;
                dd[i] *= inv_ep;
            }
            free(mog);
            free(dmul);
            free(dgo);
            free(duo);
            free(dmi);
            free(dmi2);
        }
        /* reducescatters (427-428) and the router path (431-454), per rank */
        T* wgl = (T*)calloc((size_t)(S * K), sizeof(T));
        T* dprobs = (T*)calloc((size_t)(S * N), sizeof(T));
        T* dlogits = (T*)calloc((size_t)(S * N), sizeof(T));
        T* dxr = (T*)calloc((size_t)(S * H), sizeof(T));
        const double total = (double)T_tot * (double)K;
        for (int r = 0; r < EP; ++r) {
            for (int64_t i = 0; i < S * H; ++i) {
                T acc = dgathered[r * S * H + i];
                for (int m = 1; m < EP; ++m) acc += dgathered[(int64_t)m * T_tot * H + r * S * H + i];
                dx_full[r * S * H + i] = acc;
            }
            for (int64_t i = 0; i < S * K; ++i) {
                T acc = wgrad_full[r * S * K + i];
                for (int m = 1; m < EP; ++m) acc += wgrad_full[(int64_t)m * T_tot * K + r * S * K + i];
                wgl[i] = acc;
            }
            memset(dprobs, 0, sizeof(T) * (size_t)(S * N));
            const T* pr = probs + r * S * N;
            const int64_t* ri = r_i + r * S * K;
            const T* rw = r_w + r * S * K;
            if (!fur) {
                if (c->normalize_topk) {
                    for (int64_t row = 0; row < S; ++row) {
                        double raw_sum = 0, dot = 0;
                        for (int64_t k = 0; k < K; ++k) raw_sum += (double)pr[row * N + ri[row * K + k]];
                        for (int64_t k = 0; k < K; ++k) dot += (double)wgl[row * K + k] * (double)rw[row * K + k];
                        for (int64_t k = 0; k < K; ++k)
                            dprobs[row * N + ri[row * K + k]] += (T)(((double)wgl[row * K + k] - dot) / raw_sum);
                    }
                } else {
                    for (int64_t row = 0; row < S; ++row)
                        for (int64_t k = 0; k < K; ++k) dprobs[row * N + ri[row * K + k]] += wgl[row * K + k];
                }
            }
            if (aux_coeff != 0.0) {
                /* moe.hpp:331-342 moe_aux_probs_grad */
                for (int64_t e = 0; e < N; ++e) {
                    const T v = (T)(aux_coeff * (double)N * ((double)sel[e] / total) / (double)S);
                    for (int64_t row = 0; row < S; ++row) dprobs[row * N + e] += v;
                }
            }
            SFX(softmax_backward)(pr, dprobs, dlogits, S, N);
            SFX(matmul_tn)(x_full + r * S * H, dlogits, drouter + (int64_t)r * H * N, S, H, N);
            SFX(matmul_nt)(dlogits, router, dxr, S, N, H);
            for (int64_t i = 0; i < S * H; ++i) dx_full[r * S * H + i] += dxr[i];
        }
        free(wgl);
        free(dprobs);
        free(dlogits);
        free(dxr);
    }
    for (int r = 0; r < EP; ++r) {
        for (int q = 0; q < 5; ++q) free(cache[r * 5 + q]);
        orc_artifacts_free(&arts[r]);
    }
    free(cache);
    free(arts);
    free(combined);
    free(wgrad_full);
    free(dgathered);
    free(sel);
    free(mean_probs);
    free(logits);
    free(probs);
    free(w_g);
    free(i_g);
    free(r_w);
    free(r_i);
    return 0;
}

/* moe.hpp:471-497 reference_moe_forward: the dense per-token oracle. For each token and
 * each of its K selections (k order), y = matmul(silu_glu(matmul(x, Wg_e), matmul(x, Wu_e)),
 * Wd_e) with matmul's non-f64 p-outer order (kernels.hpp:37-46) and silu_glu in fp64
 * (kernels.hpp:262-275); out[t] += w[t,k] * y. Tokens are independent (split across
 * threads); every element keeps the reference's order, so the result is bitwise its own. */
static int SFX(dense_forward)(const orc_moe_cfg* c, int64_t t_total, const T* input, const T* gate,
                              const T* up, const T* down, const T* weights, const int64_t* indices,
                              T* out) {
    const int64_t H = c->hidden, I = c->intermediate, K = c->top_k, N = c->n_experts;
    for (int64_t i = 0; i < t_total * K; ++i)
        if (indices[i] < 0 || indices[i] >= N) return 1;
#pragma omp parallel
    {
        T* g = (T*)malloc(sizeof(T) * (size_t)(3 * I + H));
        T *u = g + I, *hm = u + I, *y = hm + I;
#pragma omp for schedule(dynamic, 4)
        for (int64_t t = 0; t < t_total; ++t) {
            const T* xp = input + t * H;
            T* op = out + t * H;
            for (int64_t cc = 0; cc < H; ++cc) op[cc] = (T)0;
            for (int64_t k = 0; k < K; ++k) {
                const int64_t e = indices[t * K + k];
                const T* wg = gate + e * H * I;
                const T* wu = up + e * H * I;
                const T* wd = down + e * I * H;
                for (int64_t j = 0; j < I; ++j) g[j] = u[j] = (T)0;
                for (int64_t p = 0; p < H; ++p) {
                    const T av = xp[p];
                    for (int64_t j = 0; j < I; ++j) g[j] += av * wg[p * I + j];
                }
                for (int64_t p = 0; p < H; ++p) {
                    const T av = xp[p];
                    for (int64_t j = 0; j < I; ++j) u[j] += av * wu[p * I + j];
                }
                for (int64_t j = 0; j < I; ++j) hm[j] = (T)(SFX(silu_scalar)((double)g[j]) * (double)u[j]);
                for (int64_t cc = 0; cc < H; ++cc) y[cc] = (T)0;
                for (int64_t p = 0; p < I; ++p) {
                    const T av = hm[p];
                    for (int64_t cc = 0; cc < H; ++cc) y[cc] += av * wd[p * H + cc];
                }
                const T wv = weights[t * K + k];
                for (int64_t cc = 0; cc < H; ++cc) op[cc] += wv * y[cc];
            }
        }
        free(g);
    }
    return 0;
}
