/*
 * b2moe.h — C-ABI of the B200-native MoE expert path and EP-aware sharded AdamW.
 *
 * Drop-in boundary for the reference's hot path (arxiv 2604.00785, "Optimus";
 * reference tree /root/reference/proj). Each entry point names the reference
 * interface it replaces. All tensors are DEVICE pointers unless a parameter says
 * "host"; shapes and layouts are the reference's row-major ones:
 *   x [S,H]   router [H,N]   gate/up [NR,H,I]   down [NR,I,H]   (NR = N/EP local experts)
 * Element type per call: B2_F32 (float) or B2_BF16 (bfloat16 bits); routing
 * scores/weights are always fp32 and expert ids int64 on the host side.
 *
 * Every function returns a status: 0 ok, 1 contract violation (the reference's
 * ContractError, common.hpp:19-21), 2 bad configuration (ConfigError,
 * common.hpp:24-26), 3 CUDA error, 4 NCCL error; b2_last_error() has the message.
 * Calls are asynchronous on the context's stream unless documented otherwise.
 * There is no CPU fallback: without a B200 every compute call returns 3.
 */
#ifndef B2MOE_H
#define B2MOE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define B2_OK 0
#define B2_ERR_CONTRACT 1
#define B2_ERR_CONFIG 2
#define B2_ERR_CUDA 3
#define B2_ERR_NCCL 4
#define B2_ERR_IO 5 /* optimus::IoError: record files (reliability.cpp:272-280) */

#define B2_F32 0
#define B2_BF16 1

/* replaces optimus::MoeConfig (include/optimus/moe.hpp:13-31) */
typedef struct {
    int64_t n_experts;
    int64_t top_k;
    int64_t hidden;
    int64_t intermediate;
    int32_t ep;
    int32_t normalize_topk;
    int64_t token_block;
} b2_moe_cfg;

/* replaces optimus::AdamWConfig (include/optimus/optim.hpp:11-25) */
typedef struct {
    double beta1, beta2, eps, weight_decay, peak_lr, min_lr;
    int64_t warmup_steps, total_steps;
    double clip_norm;
    int32_t clip_after_warmup_only, round_weights_bf16;
} b2_adamw_cfg;

/* replaces optimus::ParamSlot (optim.hpp:43-49): non-owning device pointers */
typedef struct {
    void* weight;       /* [numel] weight_dtype, updated in place by b2_opt_step */
    const void* grad;   /* [numel] grad_dtype, summed over replicas by b2_opt_step */
    int64_t numel;
    int32_t cls;        /* 0 non_expert, 1 expert (optim.hpp:32-35) */
    int32_t tp_sharded;
} b2_param;

/* replaces optimus::StepStats (optim.hpp:89-94) */
typedef struct {
    int64_t step;
    double lr, grad_norm, clip_scale;
    /* B200 addition: a gradient held NaN/Inf (the soft-failure scan of
     * reliability.cpp:706-723 fused into the norm pass). As in the reference the update
     * was still applied and the step count advanced: call b2_opt_detect_soft_failure
     * before stepping, as the reference's training loop does (train.cpp:193-194) */
    int32_t nonfinite;
} b2_step_stats;

typedef struct b2_ctx b2_ctx;
typedef struct b2_moe b2_moe;
typedef struct b2_opt b2_opt;

const char* b2_last_error(void);
const char* b2_version(void);
/* 1 when the current device is an sm_100 B200 the tcgen05 kernels run on */
int b2_device_ok(void);

/* ---- rank context: replaces optimus::RankCtx (comm.hpp:205-231) --------------------
 * rank layout rank = ((pp*DP + dp)*EP + ep)*TP + tp (comm.hpp:45-59). For world > 1,
 * nccl_id is the 128-byte ncclUniqueId from b2_nccl_unique_id() on rank 0, shared
 * by the caller; the DP, EP and DPxEP communicators are split from it. `stream` is
 * the cudaStream_t every call of this context is ordered on (NULL: the legacy
 * default stream). */
int b2_nccl_unique_id(uint8_t out[128]);
int b2_ctx_create(int device, void* stream, int rank, int dp, int ep, int tp, int pp, const uint8_t* nccl_id,
                  b2_ctx** out);
int b2_ctx_destroy(b2_ctx* ctx);
int b2_ctx_sync(b2_ctx* ctx);

/* ---- FastSparseMoE layer: replaces fast_moe_forward / fast_moe_backward
 * (moe.hpp:344-466) and the state they share (FastMoeState, moe.hpp:302-316).
 * max_tokens is the per-rank S capacity; the state owns its workspace. */
int b2_moe_create(b2_ctx* ctx, const b2_moe_cfg* cfg, int dtype, int64_t max_tokens, b2_moe** out);
/* moe_block_forward's `ckpt` (blocks.cpp:339-377) and a workspace shared across layers:
 * share_workspace (or NULL) lends its activation workspace to the new layer (it must be
 * at least as large); with checkpoint != 0 the layer holds only its input pointer and the
 * balancing statistics between forward and backward, and b2_moe_backward replays the
 * forward (EP collectives included) first — gradients are bitwise those of the
 * non-checkpointed layer (test_model.cpp:680-720). The caller keeps x alive until backward. */
int b2_moe_create_ex(b2_ctx* ctx, const b2_moe_cfg* cfg, int dtype, int64_t max_tokens, const b2_moe* share_workspace,
                     int checkpoint, b2_moe** out);
/* bytes held between forward and backward (MoeRec::held, blocks.cpp:343-350) */
int64_t b2_moe_held_bytes(b2_moe* m);
int b2_moe_destroy(b2_moe* m);
/* fast_moe_forward (moe.hpp:344-390): out [S,H] */
int b2_moe_forward(b2_moe* m, const void* x, const void* router, const void* gate, const void* up,
                   const void* down, int64_t s_tokens, int fur, void* out);
/* fast_moe_backward (moe.hpp:392-466): aux_probs_grad [S,N] fp32 device or NULL;
 * expert grads come out pre-scaled by 1/EP like the reference (moe.hpp:458-461). */
int b2_moe_backward(b2_moe* m, const void* router, const void* gate, const void* up, const void* down,
                    const void* dout, const float* aux_probs_grad, void* dx, void* drouter, void* dgate,
                    void* dup, void* ddown);
/* moe_aux_probs_grad (moe.hpp:331-342) into out [S,N] fp32 device */
int b2_moe_aux_probs_grad(b2_moe* m, double coeff, float* out);
/* moe_aux_loss (moe.hpp:320-328); synchronises */
int b2_moe_aux_loss(b2_moe* m, double* out);
/* host copies of the local routing (RouteResult, moe.hpp:50-56); synchronises */
int b2_moe_routing(b2_moe* m, float* probs_host, float* weights_host, int64_t* indices_host);
/* host copies of RoutingArtifacts (moe.hpp:106-120), same field order as
 * routing_artifacts_json (moe.cpp:17-32); buffers sized for the maxima
 * (NR*TH(+1), T, T*K). sizes_host = {t_total, th, rt, padded_rows}. Synchronises. */
int b2_moe_artifacts(b2_moe* m, int64_t* sizes_host, int64_t* token_counts, int64_t* partial_token_counts,
                     int64_t* partial_cum, int64_t* cum_token_counts, int64_t* expert_counts,
                     int64_t* cum_expert_counts, int64_t* input_indices, int64_t* output_indices,
                     int64_t* selected_k, int64_t* counter);
/* MoE layer forward+backward with HOST input/output buffers (the reference's
 * Tensor-in/Tensor-out façade): x_host/dout_host -> out_host/dx_host, weights and
 * their grads device-resident. Copies run on side streams overlapped with compute.
 * Synchronises. */
int b2_moe_fwd_bwd_host(b2_moe* m, const void* x_host, const void* dout_host, const void* router,
                        const void* gate, const void* up, const void* down, double aux_coeff, void* out_host,
                        void* dx_host, void* drouter, void* dgate, void* dup, void* ddown, int64_t s_tokens);
/* Pipelined variant (B200-side addition): enqueues the same work and returns; two
 * device staging slots let step i+1's host->device copies and step i's device->host
 * results overlap the compute of the neighbouring steps. out_host/dx_host are valid
 * after b2_moe_host_wait (or a later synchronous call). Host buffers must stay alive
 * until then, and must be page-locked (cudaHostAlloc / cudaHostRegister): a pageable
 * buffer makes its copy synchronous, which serialises the pipeline (a warning is printed
 * once per handle). */
int b2_moe_fwd_bwd_host_async(b2_moe* m, const void* x_host, const void* dout_host, const void* router,
                              const void* gate, const void* up, const void* down, double aux_coeff, void* out_host,
                              void* dx_host, void* drouter, void* dgate, void* dup, void* ddown, int64_t s_tokens);
int b2_moe_host_wait(b2_moe* m);

/* ---- standalone routing stages (for identical-score parity checks) ---- */
/* route (moe.hpp:58-80): logits/probs [S,N] f32, weights [S,K] f32, indices [S,K] int32, all device */
int b2_route(b2_ctx* ctx, const b2_moe_cfg* cfg, int dtype, const void* x, const void* router, int64_t s_tokens,
             float* logits, float* probs, float* weights, int32_t* indices);
/* softmax (kernels.hpp:194-214) + topk (kernels.hpp:235-258) on given scores, device */
int b2_softmax_topk(b2_ctx* ctx, const float* logits, int64_t rows, int64_t n, int64_t k, int normalize,
                    float* probs, float* weights, int32_t* indices);
/* count_tokens + generate_indices (moe.hpp:122-197) on a device [T,K] int32 table;
 * outputs to host buffers like b2_moe_artifacts. Synchronises. */
int b2_routing_artifacts(b2_ctx* ctx, const b2_moe_cfg* cfg, const int32_t* indices, int64_t t_total, int ep_rank,
                         int64_t* sizes_host, int64_t* token_counts, int64_t* partial_token_counts,
                         int64_t* partial_cum, int64_t* cum_token_counts, int64_t* expert_counts,
                         int64_t* cum_expert_counts, int64_t* input_indices, int64_t* output_indices,
                         int64_t* selected_k, int64_t* counter);

/* ---- optimizer: replaces ShardedOptimizer (optim.hpp:98-121, optim.cpp:109-194) ---- */
#define B2_DDP 0
#define B2_SO 1
#define B2_EPSO 2
int b2_opt_create(b2_ctx* ctx, const b2_adamw_cfg* cfg, const b2_param* params, int nparams, int mode,
                  int weight_dtype, int grad_dtype, b2_opt** out);
int b2_opt_destroy(b2_opt* o);
/* ShardedOptimizer::step (optim.cpp:130-194): reduce-scatter, global norm, clip,
 * fused AdamW, all-gather. stats may be NULL (then the step does not synchronise). */
int b2_opt_step(b2_opt* o, b2_step_stats* stats);
int64_t b2_opt_state_bytes(b2_opt* o);
/* owned slice [begin,end) of param p (ShardPlan::Entry::own, optim.hpp:62-69) */
int b2_opt_owned(b2_opt* o, int p, int64_t* begin, int64_t* end);
/* host copies of the fp32 master / exp_avg / exp_avg_sq of param p's owned slice */
int b2_opt_get_state(b2_opt* o, int p, float* master, float* exp_avg, float* exp_avg_sq);
/* checkpoint assembly (reliability.cpp:411-440): the FULL fp32 master / exp_avg /
 * exp_avg_sq of param p (numel floats each, host; NULL skips one), all-gathered over the
 * param's owning group with the shard_slice bounds — collective on that group */
int b2_opt_gather_state(b2_opt* o, int p, float* master, float* exp_avg, float* exp_avg_sq);
/* restore (reliability.cpp:658-667): copy this rank's owned slice out of full host tensors */
int b2_opt_load_state(b2_opt* o, int p, const float* master, const float* exp_avg, const float* exp_avg_sq);
int b2_opt_set_step_count(b2_opt* o, int64_t n);
/* detect_soft_failure (reliability.cpp:706-723, called at train.cpp:193): NaN/Inf in
 * `loss` or in this rank's LOCAL gradients -> max over WORLD of (node + 1); *sick =
 * the highest sick node, or -1. Collective over WORLD; synchronises. */
int b2_opt_detect_soft_failure(b2_opt* o, double loss, int node, int* sick);

/* ---- sharded checkpoint record files ----
 * Format of the reference's record file (reliability.hpp:33-70, reliability.cpp:23-31):
 * "OPTT", u32 version 1, u32 count, per record {u32 name length, name, u32 dtype, u32 ndim,
 * u64 dims, little-endian payload}, u32 crc32 (zlib) of everything before it. Payloads
 * come from / go to DEVICE memory; their crc32 is computed on the GPU. */
#define B2_REC_F32 0  /* RecDtype::f32 */
#define B2_REC_BF16 1 /* RecDtype::bf16 */
typedef struct b2_rec_writer b2_rec_writer;
typedef struct b2_rec_file b2_rec_file;
/* zlib crc32(crc_in, bytes) of n DEVICE bytes (crc_in 0 starts a new checksum); synchronises */
int b2_crc32(b2_ctx* ctx, const void* dev, int64_t n, uint32_t crc_in, uint32_t* crc_out);
/* RecordFileWriter (reliability.hpp:47-71, reliability.cpp:222-270) */
int b2_rec_writer_open(b2_ctx* ctx, const char* path, b2_rec_writer** out);
/* add_f32 / add_bf16: prod(dims) elements of src_dtype (B2_F32 / B2_BF16) at DEVICE
 * pointer src; a B2_F32 source of a B2_REC_BF16 record rounds to nearest even
 * (common.hpp:116-122). Streams the payload to the file; synchronises. */
int b2_rec_writer_add(b2_rec_writer* w, const char* name, int rec_dtype, const int64_t* dims, int ndim,
                      const void* src, int src_dtype);
/* writes the header count and the crc footer, fsyncs; frees w (also on error) */
int b2_rec_writer_finish(b2_rec_writer* w, int64_t* bytes, uint32_t* crc);
/* read_record_file (reliability.cpp:272-320): validates magic, version, crc and every
 * record bound (B2_ERR_IO with the reference's message otherwise) */
int b2_rec_file_open(b2_ctx* ctx, const char* path, b2_rec_file** out);
int b2_rec_file_count(b2_rec_file* f, int* count);
/* record i: name (NUL-terminated, truncated to name_cap), dtype, dims (up to 8) */
int b2_rec_file_info(b2_rec_file* f, int i, char* name, int name_cap, int* rec_dtype, int64_t* dims, int* ndim);
int b2_rec_file_find(b2_rec_file* f, const char* name, int* index); /* -1 when absent */
/* elements [begin, end) of record i into DEVICE memory of dst_dtype (bf16 -> f32 widens) */
int b2_rec_file_read(b2_rec_file* f, int i, int64_t begin, int64_t end, void* dst, int dst_dtype);
int b2_rec_file_close(b2_rec_file* f);
/* write_state_dir's shard file (reliability.cpp:402-460): assembles the FULL master/m/v
 * of every parameter over its owning group (collective on those groups) and, on the rank
 * that is its model shard's scattered_writer (reliability.cpp:322-328), writes
 * <dir>/shard-<m>.bin with records <name>.w16 [, .master, .m, .v, .g16] for every
 * parameter the shard stores (expert, or ep coordinate 0). names[p]: record prefix;
 * dims: the shapes concatenated, ndims[p] entries each. Pass them for files the reference's
 * restore_full must read: it requires the parameter's exact shape (reliability.cpp:654);
 * dims NULL writes flat {numel} records that only this library restores.
 * full = 0: weights only. *bytes / *crc = 0 on non-writers; *model_shard = m. */
int b2_opt_write_shard(b2_opt* o, const char* dir, const char* const* names, const int64_t* dims,
                       const int* ndims, int full, int64_t* bytes, uint32_t* crc, int* model_shard);
/* restore_full's per-parameter loop (reliability.cpp:623-675): weights (and with full:
 * this rank's owned master/m/v slice and the grads) from the shard files in dir; every
 * rank reads its own files, no collective. With dims the records' shapes must match them
 * exactly (as restore_full checks); dims NULL checks element counts only. The step count
 * comes from the manifest (b2_opt_set_step_count). */
int b2_opt_restore_shard(b2_opt* o, const char* dir, const char* const* names, const int64_t* dims,
                         const int* ndims, int full);

/* adamw_update (optim.cpp:88-107) on device slices */
int b2_adamw_update(b2_ctx* ctx, float* master, float* exp_avg, float* exp_avg_sq, const void* grad,
                    int grad_dtype, int64_t n, double lr, int64_t step, const b2_adamw_cfg* cfg, void* weight_out,
                    int weight_dtype, int round_bf16);
/* replaces optimus::MemoryReport (optim.hpp:125-130) */
typedef struct {
    double weights_bytes, grads_bytes, master_bytes, optim_bytes, total_bytes, capacity_bytes;
    int32_t feasible;
} b2_memory_report_t;
/* memory_report (optim.cpp:196-221), host only: the per-device footprint of a parameter set
 * under DDP / SO / EPSO (mode 0/1/2) at DP x EP; capacity_gb is the device budget (the
 * reference's default 64 GB is a PVC tile; a B200 holds 180 GB) */
int b2_memory_report(int64_t p_expert, int64_t p_non_expert, int mode, int dp, int ep, double capacity_gb,
                     b2_memory_report_t* out);
/* lr_at_step (optim.cpp:17-24) and shard_slice (optim.cpp:43-50); host only */
double b2_lr_at_step(int64_t step, const b2_adamw_cfg* cfg);
int b2_shard_slice(int64_t numel, int group_size, int position, int64_t* begin, int64_t* end);
/* per-stage CUDA-event timing of the layer (route, index, gather, the six GEMMs,
 * combine, output-reduction backward, router backward): enable, run, then read
 * B2_MOE_NUM_STAGES floats in ms (synchronises). on: 0 off; 1 eager launches, the mean over
 * the profiled calls; 2 inside the CUDA graphs (graph mode), the last replayed call. */
#define B2_MOE_NUM_STAGES 12
int b2_moe_set_profiling(b2_moe* m, int on);
int b2_moe_stage_times(b2_moe* m, float* ms_host);
const char* b2_moe_stage_name(int stage);
/* CUDA-graph mode for b2_moe_forward / b2_moe_backward (B200-side addition; the
 * reference has no equivalent): a call whose pointer arguments and token count repeat
 * the previous call's is captured once and then replayed as a single graph launch.
 * Needs a non-default stream on the context; profiling runs eagerly. */
int b2_moe_set_graph(b2_moe* m, int on);
/* number of this library's kernels launched by the last call on the handle */
int b2_moe_last_launches(b2_moe* m);
int b2_opt_last_launches(b2_opt* o);

#ifdef __cplusplus
}
#endif
#endif /* B2MOE_H */
