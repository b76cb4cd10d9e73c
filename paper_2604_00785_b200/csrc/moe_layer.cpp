// Host orchestration of the FastSparseMoE layer on one B200 (Algorithm 1,
// include/optimus/moe.hpp:344-466), everything enqueued on the rank's stream with
// no host synchronisation inside forward/backward: data-dependent sizes (RT, the
// padded row count) stay on the device and the kernels read them from there.
//
// Stage map (reference line -> kernel):
//   route 357              router_logits + softmax_topk (+ fur_route 360-364)
//   count/indices 370-371  routing_index (count, scan, stable scatter, pad fill)
//   expert_forward 374     gather_rows; bf16: tcgen05 FwdGateUp (SwiGLU epilogue) + FwdDown
//                          fp32: SIMT gate, up, swiglu_fwd, down
//   combine 377            combine (token-major weighted K-sum)
//   stats 381-386          aux_stats
//   backward 402-454       out_reduction_bwd, dgrad/wgrad GEMMs, dx_finalize, router dW
#include "moe_layer.h"

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include <unistd.h>

#include "comm.h"
#include "kernels.h"

namespace b2 {

void MoeConfig::validate() const {
    check(n_experts >= 1 && top_k >= 1 && hidden >= 1 && intermediate >= 1 && ep >= 1,
          "moe: config fields must be positive");
    check(top_k <= n_experts, "moe: top_k cannot exceed n_experts");
    check(n_experts % ep == 0, "moe: n_experts " + std::to_string(n_experts) + " must divide evenly over ep " +
                                   std::to_string(ep));
    check(token_block >= 1, "moe: token_block must be positive");
}

Arena::~Arena() {
    if (base_ && owned_) cudaFree(base_);
}

void Arena::adopt(char* base, size_t cap) {
    check(base_ == nullptr, "arena: already reserved");
    base_ = base;
    cap_ = cap;
    off_ = 0;
    owned_ = false;
}

Workspace::~Workspace() {
    if (base) cudaFree(base);
}

void Arena::reserve(size_t bytes) {
    check(base_ == nullptr, "arena: already reserved");
    cap_ = bytes;
    B2_CUDA(cudaMalloc(&base_, std::max<size_t>(cap_, 256)));
    off_ = 0;
}

void* Arena::take_bytes(size_t bytes) {
    const size_t a = (off_ + 255) & ~size_t(255);
    check(a + bytes <= cap_, "arena: workspace exhausted");
    off_ = a + bytes;
    return base_ + a;
}

MoeLayer::MoeLayer(Context& ctx, const MoeConfig& cfg, int dtype, int64_t max_tokens, const MoeLayer* share_ws,
                   bool checkpoint)
    : ctx_(ctx), cfg_(cfg), dtype_(dtype), checkpoint_(checkpoint) {
    cfg_.validate();
    check(dtype == F32 || dtype == BF16, "moe: dtype must be f32 or bf16");
    check(cfg_.ep == ctx_.ep, "fast_moe: cfg.ep must match the EP group size");
    check(max_tokens >= 0, "moe: negative token capacity");
    const int64_t N = cfg_.n_experts, K = cfg_.top_k, H = cfg_.hidden, I = cfg_.intermediate;
    const int64_t nr = cfg_.experts_per_rank();
    smax_ = max_tokens;
    tmax_ = smax_ * cfg_.ep;  // gathered tokens (reference allgather semantics)
    pmax_ = round_up(tmax_ * std::min<int64_t>(K, nr) + nr * (kRowAlign - 1), kRowAlign);
    thmax_ = ceil_div(std::max<int64_t>(tmax_, 1), cfg_.token_block);
    const int64_t nch = ceil_div(std::max<int64_t>(tmax_, 1), 64);
    const size_t es = dtype_size(dtype);
    size_t bytes = 0;
    auto acc = [&](size_t b) { bytes += ((b + 255) & ~size_t(255)) + 256; };
    // workspace: fp32
    for (int64_t n : {smax_ * N, smax_ * N, smax_ * K, tmax_ * K, (ceil_div(smax_, 128) + 1) * N, tmax_ * K,
                      smax_ * N, (int64_t)kRouterDwMaxSplits * H * N, pmax_, pmax_ * wparts()})
        acc(4 * (size_t)std::max<int64_t>(n, 1));
    // workspace: int32
    for (int64_t n : {smax_ * K, tmax_ * K, nch * nr, nch * nr, tmax_, tmax_ + 1, nr * thmax_, nr * thmax_ + 1, nr,
                      nr + 1, nr + 1, tmax_ * K, tmax_ * K, tmax_ * K, tmax_ * K, pmax_})
        acc(4 * (size_t)std::max<int64_t>(n, 1));
    // workspace: dtype, padded rows (+ the replay output)
    for (int64_t n : {pmax_ * H, pmax_ * I, pmax_ * I, pmax_ * I, pmax_ * H, pmax_ * H, pmax_ * I, pmax_ * 2 * I,
                      pmax_ * H, smax_ * H})
        acc(es * (size_t)std::max<int64_t>(n, 1));
    acc(2 * (size_t)std::max<int64_t>(smax_ * N, 1));  // dl_bf16_
    acc(2 * (size_t)std::max<int64_t>(smax_ * N, 1));  // dl_lo_
    const int E = cfg_.ep;
    if (E > 1) {
        for (int64_t n : {tmax_ * K, tmax_ * K, smax_ * K}) acc(4 * (size_t)std::max<int64_t>(n, 1));
        acc(es * (size_t)std::max<int64_t>(smax_ * H, 1));
    }
    B2_CUDA(cudaSetDevice(ctx_.device));
    if (share_ws) {
        check(share_ws->ws_ && share_ws->ws_->cap >= bytes && share_ws->ctx_.device == ctx_.device,
              "moe: the shared workspace is too small for this layer (or on another device)");
        ws_ = share_ws->ws_;
    } else {
        ws_ = std::make_shared<Workspace>();
        B2_CUDA(cudaMalloc((void**)&ws_->base, std::max<size_t>(bytes, 256)));
        ws_->cap = bytes;
    }
    ws_arena_.adopt(ws_->base, ws_->cap);
    // persistent per-layer state
    arena_.reserve(5 * 256 + 4 * (size_t)N * 2 + 64);
    mean_probs_ = arena_.take<float>(N);
    sel_ = arena_.take<int32_t>(N);
    err_ = arena_.take<int32_t>(1);
    bar_ = arena_.take<int32_t>(8);
    colsum_ctr_ = arena_.take<int32_t>(1);
    Arena& w = ws_arena_;
    logits_ = w.take<float>(smax_ * N);
    probs_ = w.take<float>(smax_ * N);
    topw_ = w.take<float>(smax_ * K);
    fw_ = w.take<float>(tmax_ * K);
    colsum_ = w.take<float>((ceil_div(smax_, 128) + 1) * N);
    wgrad_ = w.take<float>(tmax_ * K);
    dlogits_ = w.take<float>(smax_ * N);
    dw_part_ = w.take<float>((int64_t)kRouterDwMaxSplits * H * N);
    topi_ = w.take<int32_t>(smax_ * K);
    fi_ = w.take<int32_t>(tmax_ * K);
    whist_ = w.take<int32_t>(nch * nr);
    wbase_ = w.take<int32_t>(nch * nr);
    expert_counts_ = w.take<int32_t>(tmax_);
    cec_ = w.take<int32_t>(tmax_ + 1);
    partial_counts_ = w.take<int32_t>(nr * thmax_);
    partial_cum_ = w.take<int32_t>(nr * thmax_ + 1);
    token_counts_ = w.take<int32_t>(nr);
    ctc_ = w.take<int32_t>(nr + 1);
    pad_start_ = w.take<int32_t>(nr + 1);
    input_indices_ = w.take<int32_t>(tmax_ * K);
    output_indices_ = w.take<int32_t>(tmax_ * K);
    selected_k_ = w.take<int32_t>(tmax_ * K);
    slot_prow_ = w.take<int32_t>(tmax_ * K);
    prow_src_ = w.take<int32_t>(pmax_);
    prow_w_ = w.take<float>(pmax_);
    expert_order_ = w.take<int32_t>(nr);
    wpart_ = w.take<float>(pmax_ * wparts());
    mlp_in_ = w.take_bytes(es * (size_t)std::max<int64_t>(pmax_ * H, 1));
    g_ = w.take_bytes(es * (size_t)std::max<int64_t>(pmax_ * I, 1));
    u_ = w.take_bytes(es * (size_t)std::max<int64_t>(pmax_ * I, 1));
    h_ = w.take_bytes(es * (size_t)std::max<int64_t>(pmax_ * I, 1));
    y_ = w.take_bytes(es * (size_t)std::max<int64_t>(pmax_ * H, 1));
    dy_ = w.take_bytes(es * (size_t)std::max<int64_t>(pmax_ * H, 1));
    dh_ = w.take_bytes(es * (size_t)std::max<int64_t>(pmax_ * I, 1));
    dgu_ = w.take_bytes(es * (size_t)std::max<int64_t>(pmax_ * 2 * I, 1));
    dxp_ = w.take_bytes(es * (size_t)std::max<int64_t>(pmax_ * H, 1));
    dl_bf16_ = w.take_bytes(2 * (size_t)std::max<int64_t>(smax_ * N, 1));
    dl_lo_ = w.take_bytes(2 * (size_t)std::max<int64_t>(smax_ * N, 1));
    replay_out_ = w.take_bytes(es * (size_t)std::max<int64_t>(smax_ * H, 1));
    if (E > 1) {
        check(ctx_.comm != nullptr && ctx_.comm->ep.size == E, "fast_moe: EP > 1 needs the EP communicator");
        gi_all_ = w.take<int32_t>(tmax_ * K);
        gw_all_ = w.take<float>(tmax_ * K);
        wgrad_local_ = w.take<float>(smax_ * K);
        dx_exp_ = w.take_bytes(es * (size_t)std::max<int64_t>(smax_ * H, 1));
        ep_setup();
        B2_CUDA(cudaStreamCreateWithFlags(&side_, cudaStreamNonBlocking));
        B2_CUDA(cudaEventCreateWithFlags(&ev_fork_, cudaEventDisableTiming));
        B2_CUDA(cudaEventCreateWithFlags(&ev_join_, cudaEventDisableTiming));
    }
    B2_CUDA(cudaMemsetAsync(err_, 0, 4, ctx_.stream));
    B2_CUDA(cudaMemsetAsync(colsum_ctr_, 0, 4, ctx_.stream));
    B2_CUDA(cudaMemsetAsync(pad_start_, 0, 4 * (nr + 1), ctx_.stream));
}

MoeLayer::~MoeLayer() {
    for (int i = 0; i < kGraphSlots; ++i) {
        gfwd_[i].reset();
        gbwd_[i].reset();
    }
    for (auto& st : prof_ev_)
        for (cudaEvent_t e : st) cudaEventDestroy(e);
    if (side_) {
        cudaStreamSynchronize(side_);
        cudaStreamDestroy(side_);
        cudaEventDestroy(ev_fork_);
        cudaEventDestroy(ev_join_);
    }
    if (sym_) {
        cudaStreamSynchronize(ctx_.stream);
        for (int p = 0; p < (int)peer_base_.size(); ++p)
            if (p != ctx_.coord_ep && peer_base_[(size_t)p] && peer_ipc_[(size_t)p])
                cudaIpcCloseMemHandle(peer_base_[(size_t)p]);
        cudaFree(sym_);
        cudaFree(peer_tab_);
    }
}

// symmetric buffer: [x_sh S*H | dout_sh S*H | ret_f E*S*H | ret_b E*S*H] (dtype) + wret [E*S*K] f32
// + barrier flags [E] + the published routing table [S,K] ids + weights, identical offsets on every
// rank; IPC handles are exchanged with an NCCL all-gather
void MoeLayer::ep_setup() {
    const int E = cfg_.ep, me = ctx_.coord_ep;
    const size_t es = dtype_size(dtype_);
    const size_t H = (size_t)cfg_.hidden, S = (size_t)std::max<int64_t>(smax_, 1), K = (size_t)cfg_.top_k;
    auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
    const size_t o_x = 0, o_d = o_x + al(es * S * H), o_rf = o_d + al(es * S * H), o_rb = o_rf + al(es * E * S * H),
                 o_w = o_rb + al(es * E * S * H), o_f = o_w + al(4 * E * S * K),
                 o_t = o_f + al(4 * (size_t)E), total = o_t + al(8 * S * K);
    B2_CUDA(cudaMalloc(&sym_, total));
    // barrier flags start at zero before any peer can see this buffer: the memset precedes
    // this rank's handle contribution on the same stream
    B2_CUDA(cudaMemsetAsync(sym_ + o_f, 0, 4 * (size_t)E, ctx_.stream));
    B2_CUDA(cudaMemsetAsync(bar_, 0, 4, ctx_.stream));
    // per rank: the IPC handle (other processes) plus process id, device and raw address (ranks
    // that are threads of one process — the reference's World — map peers directly instead)
    struct Pub {
        cudaIpcMemHandle_t h;
        int64_t pid;
        int64_t dev;
        uint64_t addr;
    };
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "ipc handle size");
    Pub mine{};
    B2_CUDA(cudaIpcGetMemHandle(&mine.h, sym_));
    mine.pid = (int64_t)getpid();
    mine.dev = ctx_.device;
    mine.addr = (uint64_t)(uintptr_t)sym_;
    char* dh = nullptr;
    B2_CUDA(cudaMalloc(&dh, sizeof(Pub) * (size_t)E));
    B2_CUDA(cudaMemcpyAsync(dh + sizeof(Pub) * me, &mine, sizeof(Pub), cudaMemcpyHostToDevice, ctx_.stream));
    B2_NCCL(ncclAllGather(dh + sizeof(Pub) * me, dh, sizeof(Pub), ncclUint8, ctx_.comm->ep.comm, ctx_.stream));
    std::vector<Pub> pubs((size_t)E);
    B2_CUDA(cudaMemcpyAsync(pubs.data(), dh, sizeof(Pub) * (size_t)E, cudaMemcpyDeviceToHost, ctx_.stream));
    B2_CUDA(cudaStreamSynchronize(ctx_.stream));
    B2_CUDA(cudaFree(dh));
    peer_base_.assign((size_t)E, nullptr);
    peer_ipc_.assign((size_t)E, 0);
    for (int p = 0; p < E; ++p) {
        const Pub& q = pubs[(size_t)p];
        if (p == me) {
            peer_base_[(size_t)p] = sym_;
        } else if (q.pid == mine.pid) {  // same process: direct peer access (UVA address)
            if (q.dev != ctx_.device) {
                const cudaError_t e = cudaDeviceEnablePeerAccess((int)q.dev, 0);
                if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
                else B2_CUDA(e);
            }
            peer_base_[(size_t)p] = (char*)(uintptr_t)q.addr;
        } else {
            void* ptr = nullptr;
            B2_CUDA(cudaIpcOpenMemHandle(&ptr, q.h, cudaIpcMemLazyEnablePeerAccess));
            peer_base_[(size_t)p] = (char*)ptr;
            peer_ipc_[(size_t)p] = 1;
        }
    }
    std::vector<void*> tab((size_t)8 * E);
    for (int p = 0; p < E; ++p) {
        tab[(size_t)(0 * E + p)] = peer_base_[(size_t)p] + o_x;
        tab[(size_t)(1 * E + p)] = peer_base_[(size_t)p] + o_d;
        tab[(size_t)(2 * E + p)] = peer_base_[(size_t)p] + o_rf;
        tab[(size_t)(3 * E + p)] = peer_base_[(size_t)p] + o_rb;
        tab[(size_t)(4 * E + p)] = peer_base_[(size_t)p] + o_w;
        tab[(size_t)(5 * E + p)] = peer_base_[(size_t)p] + o_f;
        tab[(size_t)(6 * E + p)] = peer_base_[(size_t)p] + o_t;                // routing ids [S,K]
        tab[(size_t)(7 * E + p)] = peer_base_[(size_t)p] + o_t + 4 * S * K;    // routing weights [S,K]
    }
    B2_CUDA(cudaMalloc(&peer_tab_, sizeof(void*) * tab.size()));
    B2_CUDA(cudaMemcpy(peer_tab_, tab.data(), sizeof(void*) * tab.size(), cudaMemcpyHostToDevice));
    x_sh_ = sym_ + o_x;
    dout_sh_ = sym_ + o_d;
    ret_f_ = sym_ + o_rf;
    ret_b_ = sym_ + o_rb;
    wret_ = (float*)(sym_ + o_w);
    flags_ = (int*)(sym_ + o_f);
    tab_ids_ = (int32_t*)(sym_ + o_t);
    tab_w_ = (float*)(sym_ + o_t + 4 * S * K);
}

// every rank's preceding stream work (and its peer stores) is complete once this returns
void MoeLayer::ep_barrier(cudaStream_t st) {
    launch_ep_flag_barrier((int* const*)peer_tab_ + 5 * cfg_.ep, flags_, bar_, cfg_.ep, ctx_.coord_ep,
                           st ? st : ctx_.stream);
}

bool MoeLayer::overlap_return() const {
    return dtype_ == BF16 && cfg_.ep >= kOverlapMinEp && side_ != nullptr && overlap_opt_;
}

const char* MoeLayer::stage_name(int s) {
    static const char* names[kNumStages] = {"route",           "index",          "gather",       "gemm_fwd_gate_up",
                                            "gemm_fwd_down",   "combine",        "out_red_bwd",  "gemm_bwd_dgrad",
                                            "gemm_wgrad_down", "gemm_wgrad_gate_up", "gemm_bwd_dx", "router_bwd"};
    return (s >= 0 && s < kNumStages) ? names[s] : "?";
}

// profiling: every forward+backward while enabled records one event pair per stage
// (up to kMaxProfSteps); stage_times() returns the mean over the recorded steps.
constexpr int kMaxProfSteps = 256;

void MoeLayer::set_profiling(int mode) {
    check(mode >= 0 && mode <= 2, "set_profiling: mode is 0, 1 or 2");
    profiling_ = mode;
    prof_step_ = -1;
    set_graph(graph_);  // graphs captured with (or without) the stage events must not be replayed
}

void MoeLayer::mark(int stage, bool end) {
    if (!profiling_ || prof_step_ < 0 || prof_step_ >= kMaxProfSteps) return;
    while ((int)prof_ev_.size() <= prof_step_) {
        std::vector<cudaEvent_t> v(2 * kNumStages);
        for (cudaEvent_t& e : v) B2_CUDA(cudaEventCreate(&e));
        prof_ev_.push_back(std::move(v));
    }
    cudaEvent_t ev = prof_ev_[(size_t)prof_step_][(size_t)(2 * stage + (end ? 1 : 0))];
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    B2_CUDA(cudaStreamIsCapturing(ctx_.stream, &cs));
    // under capture (in-graph profiling) the record becomes an event-record node of the graph
    if (cs == cudaStreamCaptureStatusActive) B2_CUDA(cudaEventRecordWithFlags(ev, ctx_.stream, cudaEventRecordExternal));
    else B2_CUDA(cudaEventRecord(ev, ctx_.stream));
}

void MoeLayer::stage_times(float* ms) {
    check(profiling_ && prof_step_ >= 0, "stage_times: no profiled step recorded");
    B2_CUDA(cudaStreamSynchronize(ctx_.stream));
    const int n = std::min(prof_step_ + 1, kMaxProfSteps);
    for (int s = 0; s < kNumStages; ++s) {
        double acc = 0;
        for (int i = 0; i < n; ++i) {
            float t = 0.f;
            B2_CUDA(cudaEventElapsedTime(&t, prof_ev_[(size_t)i][(size_t)(2 * s)], prof_ev_[(size_t)i][(size_t)(2 * s + 1)]));
            acc += t;
        }
        ms[s] = (float)(acc / n);
    }
}

void MoeLayer::GraphCache::reset() {
    if (exec) cudaGraphExecDestroy(exec);
    exec = nullptr;
    seen = false;
    key.clear();
}

void MoeLayer::set_graph(bool on) {
    B2_CUDA(cudaStreamSynchronize(ctx_.stream));
    graph_ = on;
    for (int i = 0; i < kGraphSlots; ++i) {
        gfwd_[i].reset();
        gbwd_[i].reset();
    }
}

template <typename F>
void MoeLayer::run_graphed(GraphCache (&gcs)[kGraphSlots], std::vector<const void*> key, F&& body) {
    cudaStream_t st = ctx_.stream;
    if (!graph_ || profiling_ == 1 || st == nullptr) {  // the legacy default stream cannot be captured
        body();
        return;
    }
    int& lru = graph_lru_[&gcs[0] == &gfwd_[0] ? 0 : 1];
    GraphCache* gc = nullptr;
    for (auto& c : gcs)
        if (c.seen && c.key == key) gc = &c;
    if (gc && gc->exec) {
        B2_CUDA(cudaGraphLaunch(gc->exec, st));
        launches_ = gc->launches;
        return;
    }
    if (!gc) {  // first sight of this key: run eagerly, remember it (evicting round-robin)
        gc = &gcs[lru];
        lru = (lru + 1) % kGraphSlots;
        gc->reset();
        gc->key = std::move(key);
        gc->seen = true;
        body();
        return;
    }
    cudaGraph_t g = nullptr;
    B2_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    try {
        body();
    } catch (...) {
        cudaStreamEndCapture(st, &g);
        if (g) cudaGraphDestroy(g);
        gc->reset();
        throw;
    }
    B2_CUDA(cudaStreamEndCapture(st, &g));
    const cudaError_t e = cudaGraphInstantiate(&gc->exec, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) {
        gc->reset();
        B2_CUDA(e);
    }
    gc->launches = launches_;
    B2_CUDA(cudaGraphLaunch(gc->exec, st));
}

// dispatch weights/indices of this forward (learned top-k or FUR; the gathered table at EP > 1)
void MoeLayer::set_dispatch_tables() {
    gw_ = fur_ ? (const float*)fw_ : (const float*)topw_;
    gi_ = fur_ ? (const int32_t*)fi_ : (const int32_t*)topi_;
    gi_local_ = gi_;
    if (cfg_.ep > 1) {
        gi_ = gi_all_;
        gw_ = gw_all_;
    }
}

void MoeLayer::forward(const void* x, const void* router, const void* gate, const void* up, const void* down,
                       int64_t s, bool fur, void* out) {
    check(s >= 0 && s <= smax_, "fast_moe: token count exceeds the layer's capacity");
    B2_CUDA(cudaSetDevice(ctx_.device));
    const PdlScope pdl(pdl_for_layer());
    s_ = s;
    t_ = s * cfg_.ep;
    th_ = ceil_div(std::max<int64_t>(t_, 0), cfg_.token_block);
    fur_ = fur;
    x_ = x;
    set_dispatch_tables();
    launches_ = 0;
    if (profiling_ == 1) ++prof_step_;
    else if (profiling_ == 2) prof_step_ = 0;  // in-graph: one event set, rewritten by every replay
    run_graphed(gfwd_, {x, router, gate, up, down, out, (const void*)(intptr_t)s, (const void*)(intptr_t)fur}, [&] {
        if (dtype_ == F32)
            forward_t<float>((const float*)x, (const float*)router, (const float*)gate, (const float*)up,
                             (const float*)down, fur, (float*)out);
        else
            forward_t<__nv_bfloat16>((const __nv_bfloat16*)x, (const __nv_bfloat16*)router,
                                     (const __nv_bfloat16*)gate, (const __nv_bfloat16*)up,
                                     (const __nv_bfloat16*)down, fur, (__nv_bfloat16*)out);
    });
    have_fwd_ = true;
}

template <typename T>
void MoeLayer::forward_t(const T* x, const T* router, const T* gate, const T* up, const T* down, bool fur, T* out) {
    cudaStream_t st = ctx_.stream;
    const int E = cfg_.ep;
    const int S = (int)s_, N = (int)cfg_.n_experts, K = (int)cfg_.top_k, H = (int)cfg_.hidden,
              I = (int)cfg_.intermediate, nr = (int)cfg_.experts_per_rank();
    int Tt = S;  // rows of the (gathered) table this rank processes
    // stage 1: route locally (moe.hpp:357-364)
    mark(kRoute, false);
    launch_router_logits<T>(x, router, logits_, S, H, N, st);
    launch_softmax_topk(logits_, probs_, topw_, topi_, S, N, K, cfg_.normalize_topk, st);
    launches_ += 2;
    if (fur) {
        launch_fur_route(fw_, fi_, S, N, K, st);
        launches_ += 1;
    }
    if (E > 1) {
        // the allgathers of weights and indices (moe.hpp:366-367): the reference's gathered
        // routing table; token rows stay where they are until an expert owner pulls them.
        // Publish x and this rank's table in the symmetric buffer, barrier, then pull every
        // rank's table (NVLink peer memory; no NCCL on the step's path)
        B2_CUDA(cudaMemcpyAsync(x_sh_, x, sizeof(T) * (size_t)S * H, cudaMemcpyDeviceToDevice, st));
        B2_CUDA(cudaMemcpyAsync(tab_ids_, gi_local_, 4 * (size_t)S * K, cudaMemcpyDeviceToDevice, st));
        B2_CUDA(cudaMemcpyAsync(tab_w_, fur ? (const float*)fw_ : (const float*)topw_, 4 * (size_t)S * K,
                                cudaMemcpyDeviceToDevice, st));
        ep_barrier();
        launch_ep_table_pull((const int32_t* const*)peer_tab_ + 6 * E, (const float* const*)peer_tab_ + 7 * E,
                             (int64_t)S * K, E, gi_all_, gw_all_, st);
        launches_ += 2;
        Tt = E * S;
    }
    // balancing statistics (381-386): mean_probs over the local rows, sel_counts over the
    // gathered table
    launch_aux_stats(probs_, S, N, gi_, (int64_t)Tt * K, colsum_, colsum_ctr_, mean_probs_, sel_, st);
    launches_ += 2;
    mark(kRoute, true);
    mark(kIndex, false);
    // stages 2+3 (370-371)
    RoutingIndexArgs ra{};
    ra.gidx = gi_;
    ra.T = Tt;
    ra.K = K;
    ra.N = N;
    ra.n_start = ctx_.coord_ep * nr;
    ra.nr = nr;
    ra.whist = whist_;
    ra.wbase = wbase_;
    ra.expert_counts = expert_counts_;
    ra.cum_expert_counts = cec_;
    ra.token_counts = token_counts_;
    ra.cum_token_counts = ctc_;
    ra.pad_start = pad_start_;
    ra.input_indices = input_indices_;
    ra.output_indices = output_indices_;
    ra.selected_k = selected_k_;
    ra.slot_prow = slot_prow_;
    ra.prow_src = prow_src_;
    ra.gw = gw_;
    ra.prow_w = dtype_ == BF16 ? prow_w_ : nullptr;  // weighted-H scheme of the tensor-core path
    ra.err = err_;
    ra.expert_order = dtype_ == BF16 ? expert_order_ : nullptr;  // wgrad tile order
    launch_routing_index(ra, st);
    launches_ += 4;
    mark(kIndex, true);
    const int32_t* p_total = pad_start_ + nr;
    // stage 4: expert MLP over the padded expert-sorted rows (225-244)
    mark(kGather, false);
    if (E > 1) {
        launch_ep_gather_pull<T>((const T* const*)peer_tab_, S, Tt, H, cec_, slot_prow_, (T*)mlp_in_, st);
        launch_zero_pad_rows<T>((T*)mlp_in_, prow_src_, p_total, H, pmax_, st);
        launches_ += 2;
    } else {
        launch_gather_tokens<T>(x, cec_, slot_prow_, S, prow_src_, p_total, (T*)mlp_in_, H, pmax_, st);
        launches_ += 1;
    }
    mark(kGather, true);
    if (dtype_ == BF16) {
        Sm100GemmArgs ga{};
        ga.H = H;
        ga.I = I;
        ga.nr = nr;
        ga.pmax = pmax_;
        ga.pad_start = pad_start_;
        ga.counts = token_counts_;
        ga.num_sms = ctx_.num_sms;
        ga.kind = GemmKind::FwdGateUp;
        ga.x = mlp_in_;
        ga.wg = gate;
        ga.wu = up;
        ga.out0 = g_;
        ga.out1 = u_;
        ga.out2 = h_;  // H' = w * silu(G) * U (weighted-H scheme: row_w)
        ga.row_w = prow_w_;
        mark(kGemmGateUp, false);
        launch_sm100_gemm(ga, st);
        mark(kGemmGateUp, true);
        ga.kind = GemmKind::FwdDown;
        ga.h = h_;
        ga.wd = down;
        ga.out0 = y_;
        mark(kGemmDown, false);
        launch_sm100_gemm(ga, st);
        mark(kGemmDown, true);
        launches_ += 2;
    } else {
        SimtGemmArgs a{};
        a.group_start = pad_start_;
        a.groups = nr;
        a.by_k = 0;
        a.M_lim = pmax_;
        a.scale = 1.f;
        // G = X . Wg, U = X . Wu   (A [P,H] K-major; B [H,I] per expert)
        a.A = mlp_in_;
        a.lda_m = H;
        a.lda_k = 1;
        a.ldb_k = I;
        a.ldb_n = 1;
        a.b_gs = (int64_t)H * I;
        a.ldd_m = I;
        a.ldd_n = 1;
        a.N = I;
        a.K = H;
        a.B = gate;
        a.D = g_;
        mark(kGemmGateUp, false);
        launch_simt_grouped_gemm<T>(a, pmax_, st);
        a.B = up;
        a.D = u_;
        launch_simt_grouped_gemm<T>(a, pmax_, st);
        launch_swiglu_fwd<T>((const T*)g_, (const T*)u_, (T*)h_, p_total, I, pmax_, st);
        mark(kGemmGateUp, true);
        mark(kGemmDown, false);
        // Y = H . Wd
        a.A = h_;
        a.lda_m = I;
        a.ldb_k = H;
        a.b_gs = (int64_t)I * H;
        a.ldd_m = H;
        a.N = H;
        a.K = I;
        a.B = down;
        a.D = y_;
        launch_simt_grouped_gemm<T>(a, pmax_, st);
        mark(kGemmDown, true);
        launches_ += 4;
    }
    // stage 5: weighted combine (377); EP = 1 so the reducescatter (378) is the identity
    mark(kCombine, false);
    if (E > 1) {
        // each owner combines its slots into its OWN slab row [gid]; after the barrier the
        // source pulls its rows from the owners and sums them in rank order
        // bf16: the rows are already weighted (y' = H' . Wd = w * y), fp32: weight here
        launch_ep_combine_local<T>((const T*)y_, slot_prow_, selected_k_, cec_, dtype_ == BF16 ? nullptr : gw_, K, S,
                                   Tt, H, (T*)ret_f_, st, 0, (T* const*)peer_tab_ + 2 * E, ctx_.coord_ep);
        ep_barrier();
        launch_ep_pull_sum<T>((const T* const*)peer_tab_ + 2 * E, gi_local_, S, K, E, nr, H, ctx_.coord_ep, out, st, 0,
                              true);
        launches_ += 2;
    } else {
        launch_combine<T>((const T*)y_, slot_prow_, selected_k_, cec_, dtype_ == BF16 ? nullptr : gw_, out, Tt, H, K,
                          st);
        launches_ += 1;
    }
    mark(kCombine, true);
}

void MoeLayer::backward(const void* router, const void* gate, const void* up, const void* down, const void* dout,
                        const float* aux_probs_grad, void* dx, void* drouter, void* dgate, void* dup, void* ddown) {
    check(have_fwd_, "fast_moe_backward: no forward state");
    B2_CUDA(cudaSetDevice(ctx_.device));
    const PdlScope pdl(pdl_for_layer());
    launches_ = 0;
    run_graphed(gbwd_,
                {router, gate, up, down, dout, aux_probs_grad, dx, drouter, dgate, dup, ddown, x_,
                 (const void*)(intptr_t)s_, (const void*)(intptr_t)fur_},
                [&] {
                    if (checkpoint_) {
                        // moe_block_backward with ckpt (blocks.cpp:361-367): replay the forward,
                        // its EP collectives included, from the held input; deterministic
                        // kernels make the replayed state bitwise equal to the original
                        if (dtype_ == F32)
                            forward_t<float>((const float*)x_, (const float*)router, (const float*)gate,
                                             (const float*)up, (const float*)down, fur_, (float*)replay_out_);
                        else
                            forward_t<__nv_bfloat16>((const __nv_bfloat16*)x_, (const __nv_bfloat16*)router,
                                                     (const __nv_bfloat16*)gate, (const __nv_bfloat16*)up,
                                                     (const __nv_bfloat16*)down, fur_, (__nv_bfloat16*)replay_out_);
                    }
                    if (dtype_ == F32)
                        backward_t<float>((const float*)router, (const float*)gate, (const float*)up,
                                          (const float*)down, (const float*)dout, aux_probs_grad, (float*)dx,
                                          (float*)drouter, (float*)dgate, (float*)dup, (float*)ddown);
                    else
                        backward_t<__nv_bfloat16>(
                            (const __nv_bfloat16*)router, (const __nv_bfloat16*)gate, (const __nv_bfloat16*)up,
                            (const __nv_bfloat16*)down, (const __nv_bfloat16*)dout, aux_probs_grad,
                            (__nv_bfloat16*)dx, (__nv_bfloat16*)drouter, (__nv_bfloat16*)dgate,
                            (__nv_bfloat16*)dup, (__nv_bfloat16*)ddown);
                });
}

template <typename T>
void MoeLayer::backward_t(const T* router, const T* gate, const T* up, const T* down, const T* dout,
                          const float* aux_probs_grad, T* dx, T* drouter, T* dgate, T* dup, T* ddown) {
    cudaStream_t st = ctx_.stream;
    const int E = cfg_.ep;
    const int S = (int)s_, Tt = (int)t_, N = (int)cfg_.n_experts, K = (int)cfg_.top_k, H = (int)cfg_.hidden,
              I = (int)cfg_.intermediate, nr = (int)cfg_.experts_per_rank();
    const int32_t* p_total = pad_start_ + nr;
    const float inv_ep = (float)(1.0 / (double)cfg_.ep);
    // output_reduction_backward (402-403). The allgather of dout (400) becomes a dispatch of
    // dout rows to the same ranks the tokens went to.
    mark(kOutRedBwd, false);
    const T* const* peer_dout = nullptr;
    if (E > 1) {  // owners pull dout rows straight from the source rank
        B2_CUDA(cudaMemcpyAsync(dout_sh_, dout, sizeof(T) * (size_t)S * H, cudaMemcpyDeviceToDevice, st));
        ep_barrier();
        peer_dout = (const T* const*)peer_tab_ + E;
    }
    // EP > 1: the top-k weight gradients go straight into this rank's symmetric slab, where
    // the sources pull them from
    if (dtype_ == BF16) {
        // weighted-H scheme: dY is just the token's dout row in each of its padded rows (the
        // routing weight is applied inside the dgrad epilogue, and the weight gradient comes out
        // of that epilogue's dot products) — a plain gather, no mlp_out read
        if (E > 1) {
            launch_ep_gather_pull<T>(peer_dout, S, Tt, H, cec_, slot_prow_, (T*)dy_, st);
            launch_zero_pad_rows<T>((T*)dy_, prow_src_, p_total, H, pmax_, st);
            launches_ += 2;
        } else {
            launch_gather_tokens<T>(dout, cec_, slot_prow_, S, prow_src_, p_total, (T*)dy_, H, pmax_, st);
            launches_ += 1;
        }
    } else {
        launch_out_reduction_bwd<T>(dout, peer_dout, S, (const T*)y_, slot_prow_, selected_k_, cec_, gw_, (T*)dy_,
                                    E > 1 ? wret_ : wgrad_, Tt, H, K, st);
        launch_zero_pad_rows<T>((T*)dy_, prow_src_, p_total, H, pmax_, st);
        launches_ += 2;
    }
    mark(kOutRedBwd, true);
    if (dtype_ == BF16) {
        Sm100GemmArgs ga{};
        ga.H = H;
        ga.I = I;
        ga.nr = nr;
        ga.pmax = pmax_;
        ga.pad_start = pad_start_;
        ga.counts = token_counts_;
        ga.num_sms = ctx_.num_sms;
        ga.x = mlp_in_;
        ga.wg = gate;
        ga.wu = up;
        ga.wd = down;
        ga.expert_order = expert_order_;
        ga.g = g_;
        ga.u = u_;
        ga.h = h_;
        ga.dy = dy_;
        ga.dgu = dgu_;
        ga.scale = inv_ep;
        ga.kind = GemmKind::BwdDownDgrad;  // 406 + silu_glu_backward 409
        ga.out0 = dgu_;
        ga.row_w = prow_w_;
        ga.wpart = wpart_;
        mark(kGemmDgrad, false);
        launch_sm100_gemm(ga, st);
        ga.row_w = nullptr;
        ga.wpart = nullptr;
        launch_wgrad_from_parts(wpart_, (int)wparts(), slot_prow_, selected_k_, cec_, E > 1 ? wret_ : wgrad_, Tt, K,
                                st);
        launches_ += 1;
        mark(kGemmDgrad, true);
        if (overlap_return()) {
            // EP > 1: dX first, then its return to the source ranks (owner combine pushed into
            // the sources' slabs, barrier, rank-order sums: the reducescatters of moe.hpp:427-428)
            // runs on a side stream
            // while the weight-gradient GEMMs run on the SMs left to them
            ga.kind = GemmKind::BwdDx;  // 414-415
            ga.out0 = dxp_;
            mark(kGemmDx, false);
            launch_sm100_gemm(ga, st);
            mark(kGemmDx, true);
            B2_CUDA(cudaEventRecord(ev_fork_, st));
            B2_CUDA(cudaStreamWaitEvent(side_, ev_fork_, 0));
            // side-stream grids capped to the reserved SMs (8 resident 256-thread blocks each), so
            // they never hold SMs the weight-gradient GEMM's CTAs are waiting for
            const int side_cap = kCommSms * 8;
            launch_ep_combine_local<T>((const T*)dxp_, slot_prow_, selected_k_, cec_, nullptr, K, S, Tt, H,
                                       (T*)ret_b_, side_, side_cap, (T* const*)peer_tab_ + 3 * E, ctx_.coord_ep);
            ep_barrier(side_);
            launch_ep_pull_sum<T>((const T* const*)peer_tab_ + 3 * E, gi_local_, S, K, E, nr, H, ctx_.coord_ep,
                                  (T*)dx_exp_, side_, side_cap, true);
            launch_ep_pull_sum<float>((const float* const*)peer_tab_ + 4 * E, gi_local_, S, K, E, nr, K,
                                      ctx_.coord_ep, wgrad_local_, side_, side_cap);
            B2_CUDA(cudaEventRecord(ev_join_, side_));
            ga.max_ctas = ctx_.num_sms - kCommSms;
        }
        ga.kind = GemmKind::WgradDown;  // 407
        ga.out0 = ddown;
        mark(kGemmWgradDown, false);
        launch_sm100_gemm(ga, st);
        mark(kGemmWgradDown, true);
        ga.kind = GemmKind::WgradGateUp;  // 410-413
        ga.out0 = dgate;
        ga.out1 = dup;
        mark(kGemmWgradGateUp, false);
        launch_sm100_gemm(ga, st);
        mark(kGemmWgradGateUp, true);
        ga.max_ctas = 0;
        if (overlap_return()) {
            B2_CUDA(cudaStreamWaitEvent(st, ev_join_, 0));
            launches_ += 4 + 4;
        } else {
            ga.kind = GemmKind::BwdDx;  // 414-415
            ga.out0 = dxp_;
            mark(kGemmDx, false);
            launch_sm100_gemm(ga, st);
            mark(kGemmDx, true);
            launches_ += 4;
        }
    } else {
        SimtGemmArgs a{};
        a.group_start = pad_start_;
        a.groups = nr;
        a.scale = 1.f;
        // dH = dY . Wd^T (grouped_mm_nt): A [P,H]; B(k=h, n=i) = Wd[e][i][h]
        a.by_k = 0;
        a.M_lim = pmax_;
        a.A = dy_;
        a.lda_m = H;
        a.lda_k = 1;
        a.B = down;
        a.ldb_k = 1;
        a.ldb_n = H;
        a.b_gs = (int64_t)I * H;
        a.D = dh_;
        a.ldd_m = I;
        a.ldd_n = 1;
        a.N = I;
        a.K = H;
        mark(kGemmDgrad, false);
        launch_simt_grouped_gemm<T>(a, pmax_, st);
        launch_swiglu_bwd<T>((const T*)g_, (const T*)u_, (const T*)dh_, (T*)dgu_, p_total, I, pmax_, st);
        // dWd[e] = H^T . dY over the rows of e, scaled 1/EP (407, 458-461)
        SimtGemmArgs w{};
        w.group_start = pad_start_;
        w.groups = nr;
        w.by_k = 1;
        w.scale = inv_ep;
        w.A = h_;
        w.lda_m = 1;
        w.lda_k = I;
        w.B = dy_;
        w.ldb_k = H;
        w.ldb_n = 1;
        w.D = ddown;
        w.ldd_m = H;
        w.ldd_n = 1;
        w.d_gs = (int64_t)I * H;
        w.M_lim = I;
        w.N = H;
        mark(kGemmDgrad, true);
        mark(kGemmWgradDown, false);
        launch_simt_grouped_gemm<T>(w, I, st);
        mark(kGemmWgradDown, true);
        mark(kGemmWgradGateUp, false);
        // dWg[e] = X^T . dG, dWu[e] = X^T . dU (410-413)
        w.A = mlp_in_;
        w.lda_k = H;
        w.B = dgu_;
        w.ldb_k = 2 * I;
        w.D = dgate;
        w.ldd_m = I;
        w.d_gs = (int64_t)H * I;
        w.M_lim = H;
        w.N = I;
        launch_simt_grouped_gemm<T>(w, H, st);
        w.B = (const T*)dgu_ + I;
        w.D = dup;
        launch_simt_grouped_gemm<T>(w, H, st);
        mark(kGemmWgradGateUp, true);
        mark(kGemmDx, false);
        // dX_perm = dG . Wg^T + dU . Wu^T (414-415)
        a.A = dgu_;
        a.lda_m = 2 * I;
        a.B = gate;
        a.ldb_k = 1;
        a.ldb_n = I;
        a.b_gs = (int64_t)H * I;
        a.D = dxp_;
        a.ldd_m = H;
        a.N = H;
        a.K = I;
        launch_simt_grouped_gemm<T>(a, pmax_, st);
        a.A = (const T*)dgu_ + I;
        a.B = up;
        a.accumulate = 1;
        launch_simt_grouped_gemm<T>(a, pmax_, st);
        mark(kGemmDx, true);
        launches_ += 7;
    }
    // router path (431-454)
    mark(kRouterBwd, false);
    const float* wgrad_local = wgrad_;
    const T* dx_rows = nullptr;  // EP > 1: the token's summed expert-gradient rows
    if (E > 1 && overlap_return()) {  // already returned on the side stream
        wgrad_local = wgrad_local_;
        dx_rows = (const T*)dx_exp_;
    } else if (E > 1) {
        // the two reducescatters of moe.hpp:427-428: owners combine dX partials and push them
        // into the sources' slabs (the top-k weight gradients already sit in the owners' wret);
        // after the barrier each source sums its dX rows and pulls and sums its weight
        // gradients, in rank order
        launch_ep_combine_local<T>((const T*)dxp_, slot_prow_, selected_k_, cec_, nullptr, K, S, Tt, H, (T*)ret_b_,
                                   st, 0, (T* const*)peer_tab_ + 3 * E, ctx_.coord_ep);
        ep_barrier();
        launch_ep_pull_sum<T>((const T* const*)peer_tab_ + 3 * E, gi_local_, S, K, E, nr, H, ctx_.coord_ep,
                              (T*)dx_exp_, st, 0, true);
        launch_ep_pull_sum<float>((const float* const*)peer_tab_ + 4 * E, gi_local_, S, K, E, nr, K, ctx_.coord_ep,
                                  wgrad_local_, st);
        wgrad_local = wgrad_local_;
        dx_rows = (const T*)dx_exp_;
        launches_ += 3;
    }
    const bool tc_router = dtype_ == BF16 && N % 8 == 0 && N <= 256;
    launch_router_dlogits(probs_, wgrad_local, topi_, topw_, aux_probs_grad, dlogits_, tc_router ? dl_bf16_ : nullptr,
                          tc_router ? dl_lo_ : nullptr, S, N, K, cfg_.normalize_topk, fur_, st);
    if (tc_router) {
        // router dW and dx on the tensor cores (fp32 accumulation; dW from bf16 dlogits, dx from the
        // two-term hi + lo split so the O(1) router weights of a real model keep dx fp32-accurate)
        Sm100GemmArgs ga{};
        ga.H = H;
        ga.I = I;
        ga.nr = 1;
        ga.pmax = pmax_;
        ga.pad_start = pad_start_;
        ga.num_sms = ctx_.num_sms;
        ga.S = S;
        ga.N = N;
        ga.x = x_;
        ga.dl = dl_bf16_;
        ga.dl_lo = dl_lo_;
        ga.wr = router;
        ga.part = dw_part_;
        ga.kind = GemmKind::RouterDw;
        launch_sm100_gemm(ga, st);
        launch_router_dw_reduce_bf16(dw_part_, drouter, router_dw_splits(S, H, ctx_.num_sms), (int64_t)H * N, st);
        // scatter-add to tokens (418-423), then + matmul_nt(dlogits, router) (454) as a GEMM whose
        // epilogue adds the scattered rows. EP = 1: a combine kernel sums each token's slot rows of
        // dXperm first (gathering them inside the RouterDx epilogue measured slower: 5.08-5.12 vs
        // 4.85 ms per step, too few bytes in flight per one-CTA tile)
        if (!dx_rows) {
            launch_combine<T>((const T*)dxp_, slot_prow_, selected_k_, cec_, nullptr, dx, S, H, K, st);
            dx_rows = dx;
        }
        ga.kind = GemmKind::RouterDx;
        ga.src = dx_rows;
        ga.out0 = dx;
        launch_sm100_gemm(ga, st);
        launches_ += 5;
    } else {
        launch_router_dw<T>((const T*)x_, dlogits_, drouter, dw_part_, kRouterDwMaxSplits, S, H, N, st);
        // scatter-add to tokens (418-423) + matmul_nt(dlogits, router) (454)
        if (dx_rows)
            launch_dx_finalize<T>(dx_rows, false, slot_prow_, cec_, dlogits_, router, dx, S, H, N, st);
        else
            launch_dx_finalize<T>((const T*)dxp_, true, slot_prow_, cec_, dlogits_, router, dx, S, H, N, st);
        launches_ += 4;
    }
    mark(kRouterBwd, true);
}

size_t MoeLayer::held_bytes() const {
    const size_t persistent = arena_.used();
    return checkpoint_ ? persistent + (size_t)s_ * (size_t)cfg_.hidden * dtype_size(dtype_)  // + the input
                       : persistent + ws_arena_.used();
}

void MoeLayer::aux_probs_grad(double coeff, float* out) {
    check(have_fwd_, "moe_aux_probs_grad: no forward state");
    const double total = (double)t_ * (double)cfg_.top_k;
    launch_aux_probs_grad(sel_, out, (int)s_, (int)cfg_.n_experts, coeff, total, ctx_.stream);
}

// count_tokens throws on an expert id outside [0, N) (moe.hpp:143-146). The index kernels flag
// it on the device without a host sync; the layer's synchronising readbacks (aux loss,
// artifacts) surface it — the flag is sticky until read, so a bad id in any forward since the
// last readback (e.g. a corrupt table pulled from a peer at EP > 1) raises here.
void MoeLayer::check_expert_ids() {
    int32_t bad = 0;
    B2_CUDA(cudaMemcpyAsync(&bad, err_, 4, cudaMemcpyDeviceToHost, ctx_.stream));
    B2_CUDA(cudaStreamSynchronize(ctx_.stream));
    if (bad) {
        B2_CUDA(cudaMemsetAsync(err_, 0, 4, ctx_.stream));
        check(false, "count_tokens: expert id out of range [0," + std::to_string(cfg_.n_experts) +
                         ") in a routing table of this layer");
    }
}

double MoeLayer::aux_loss() {
    check(have_fwd_, "moe_aux_loss: no forward state");
    check_expert_ids();
    const int N = (int)cfg_.n_experts;
    std::vector<float> mp(N);
    std::vector<int32_t> sel(N);
    B2_CUDA(cudaMemcpyAsync(mp.data(), mean_probs_, 4 * N, cudaMemcpyDeviceToHost, ctx_.stream));
    B2_CUDA(cudaMemcpyAsync(sel.data(), sel_, 4 * N, cudaMemcpyDeviceToHost, ctx_.stream));
    B2_CUDA(cudaStreamSynchronize(ctx_.stream));
    const double total = (double)t_ * (double)cfg_.top_k;
    double acc = 0;
    for (int e = 0; e < N; ++e) acc += ((double)sel[e] / total) * (double)mp[e];
    return (double)N * acc;
}

static std::vector<int64_t> d2h_i64(const int32_t* d, int64_t n, cudaStream_t st) {
    std::vector<int32_t> tmp((size_t)std::max<int64_t>(n, 0));
    if (n > 0) B2_CUDA(cudaMemcpyAsync(tmp.data(), d, 4 * (size_t)n, cudaMemcpyDeviceToHost, st));
    B2_CUDA(cudaStreamSynchronize(st));
    return std::vector<int64_t>(tmp.begin(), tmp.end());
}

MoeLayer::HostArtifacts MoeLayer::artifacts() {
    check(have_fwd_, "artifacts: no forward state");
    check_expert_ids();
    cudaStream_t st = ctx_.stream;
    const int64_t nr = cfg_.experts_per_rank(), K = cfg_.top_k, tbs = cfg_.token_block;
    HostArtifacts a;
    a.t_total = t_;
    a.th = th_;
    a.cum_token_counts = d2h_i64(ctc_, nr + 1, st);
    a.rt = a.cum_token_counts[(size_t)nr];
    a.pad_start = d2h_i64(pad_start_, nr + 1, st);
    a.padded_rows = a.pad_start[(size_t)nr];
    a.token_counts = d2h_i64(token_counts_, nr, st);
    a.input_indices = d2h_i64(input_indices_, a.rt, st);
    a.output_indices = d2h_i64(output_indices_, a.rt, st);
    a.selected_k = d2h_i64(selected_k_, a.rt, st);
    launch_partial_counts(gi_, (int)t_, (int)K, ctx_.coord_ep * (int)nr, (int)nr, (int)tbs, (int)th_, partial_counts_,
                          partial_cum_, st);
    a.partial_token_counts = d2h_i64(partial_counts_, nr * th_, st);
    a.partial_cum = d2h_i64(partial_cum_, nr * th_ + 1, st);
    a.expert_counts = d2h_i64(expert_counts_, t_, st);
    a.cum_expert_counts = d2h_i64(cec_, t_ + 1, st);
    // final write cursors of generate_indices (moe.hpp:176-188): partial_cum[ln*TH + tid + 1]
    a.counter.resize((size_t)(nr * th_));
    for (int64_t i = 0; i < nr * th_; ++i) a.counter[(size_t)i] = a.partial_cum[(size_t)i + 1];
    return a;
}

void MoeLayer::routing(float* probs, float* weights, int64_t* indices) {
    check(have_fwd_, "routing: no forward state");
    cudaStream_t st = ctx_.stream;
    const int64_t N = cfg_.n_experts, K = cfg_.top_k;
    if (probs) B2_CUDA(cudaMemcpyAsync(probs, probs_, 4 * (size_t)(s_ * N), cudaMemcpyDeviceToHost, st));
    if (weights) B2_CUDA(cudaMemcpyAsync(weights, topw_, 4 * (size_t)(s_ * K), cudaMemcpyDeviceToHost, st));
    if (indices) {
        std::vector<int64_t> v = d2h_i64(topi_, s_ * K, st);
        std::memcpy(indices, v.data(), 8 * v.size());
    }
    B2_CUDA(cudaStreamSynchronize(st));
}

void MoeLayer::mean_probs_sel(float* mean_probs, int64_t* sel_counts) {
    cudaStream_t st = ctx_.stream;
    const int64_t N = cfg_.n_experts;
    if (mean_probs) B2_CUDA(cudaMemcpyAsync(mean_probs, mean_probs_, 4 * (size_t)N, cudaMemcpyDeviceToHost, st));
    if (sel_counts) {
        std::vector<int64_t> v = d2h_i64(sel_, N, st);
        std::memcpy(sel_counts, v.data(), 8 * v.size());
    }
    B2_CUDA(cudaStreamSynchronize(st));
}

}  // namespace b2
