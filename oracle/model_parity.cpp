// TEST INFRASTRUCTURE ONLY — the model-level integration check of SURVEY §8(f)3.
//
// One serial training pass of the UNMODIFIED reference model: the multi-rank equivalence
// config of test_model.cpp:86-99 (4 layers, hidden 32, 4 x 8 heads, 4 experts top-2, ffn 48,
// vocab 64, context 8, aux coeff 0.01), batch random_tokens(8, 8, 64, 8000)
// (test_model.cpp:19-24), seed 23, gpipe with M microbatches, through pp_forward_backward
// (model.cpp:271-382 chunk_forward / chunk_backward inside). Built twice by oracle/Makefile:
//   model_parity_ref  as is (every MoE block on the reference's fast_moe_forward/backward)
//   model_parity_gpu  linked with model_gpu_adapter.cpp and -Wl,--wrap on moe_block_forward /
//                     moe_block_backward: every MoE block on the B200 (libb2moe.so)
// Output (argv[1]): "<ce_sum> <aux_sum> <n_slots>\n" then per slot "<name> <numel>\n" and the
// gradient as raw float32. With argv[3] = K > 0 the pass is K end-to-end train_step calls instead
// (model.cpp:538-565: forward/backward + the reference's EPSO AdamW step, warmup 0; with
// B2_ADAPTER_GPU_OPT=1 the GPU build runs that step on the B200 too): the header carries the K
// per-step losses and the slots hold the final weights.
// argv[4] = "wide": hidden 128, 4 x 32 heads, 8 experts of ffn 128 (the bf16 layer's shapes).
// argv[5] = EP: that many rank threads (Topology{ep}), each on the strided rows of
// test_model.cpp:30-37 and (GPU build) on the GPU of its EP coordinate; one output file per rank.
// tests/test_gpu_model_parity.py compares the two builds.
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "optimus/comm.hpp"
#include "optimus/model.hpp"
#include "optimus/optim.hpp"
#include "optimus/schedule.hpp"

using namespace optimus;

// model_gpu_adapter.cpp (model_parity_gpu only): route ShardedOptimizer::step to the B200
void b2_adapter_use_gpu_optimizer(const std::vector<ParamSlot>& slots, const AdamWConfig& c) __attribute__((weak));

int main(int argc, char** argv) {
    if (argc < 2) {
        std::fprintf(stderr, "usage: %s out.bin [microbatches]\n", argv[0]);
        return 2;
    }
    const int m = argc > 2 ? std::atoi(argv[2]) : 1;
    const int steps = argc > 3 ? std::atoi(argv[3]) : 0;
    ModelConfig cfg;
    cfg.layers = 4;
    cfg.hidden = 32;
    cfg.heads = 4;
    cfg.head_size = 8;
    cfg.intermediate = 48;
    cfg.experts = 4;
    cfg.top_k = 2;
    cfg.vocab = 64;
    cfg.context = 8;
    cfg.aux_loss_coeff = 0.01;
    if (argc > 4 && std::string(argv[4]) == "wide") {  // dims the bf16 tensor-core layer takes (H, I % 64 == 0)
        cfg.hidden = 128;
        cfg.heads = 4;
        cfg.head_size = 32;
        cfg.intermediate = 128;
        cfg.experts = 8;
    }
    TensorI batch({8, cfg.context});
    for (int64_t i = 0; i < batch.numel(); ++i) batch.data()[i] = (int64_t)(hash_mix(8000, (uint64_t)i) % (uint64_t)cfg.vocab);
    const int ep = argc > 5 ? std::atoi(argv[5]) : 1;  // EP ranks (threads of the reference's World)
    Topology serial;
    serial.ep = ep;
    World w(serial);
    int rc = 0;
    w.run([&](RankCtx& ctx) {
        Model mdl(cfg, serial, ctx.coord(), 23, 1);
        PipelineSchedule sched = pp_build_schedule(ScheduleKind::gpipe, 1, m, 1);
        ActLedger led;
        std::vector<double> losses;
        PpLossParts parts;
        // strided rows per EP replica (test_model.cpp:30-37)
        const int64_t rows = batch.dim(0) / ep, c = batch.dim(1);
        TensorI local({rows, c});
        for (int64_t r = 0; r < rows; ++r)
            for (int64_t j = 0; j < c; ++j) local.data()[r * c + j] = batch.data()[(r * ep + ctx.coord().ep) * c + j];
        if (steps > 0) {
            AdamWConfig ac;
            ac.warmup_steps = 0;
            ShardedOptimizer opt(ctx, ac, mdl.param_slots(), ShardMode::epso);
            const char* gopt = std::getenv("B2_ADAPTER_GPU_OPT");
            if (gopt && std::atoi(gopt) == 1 && b2_adapter_use_gpu_optimizer)
                b2_adapter_use_gpu_optimizer(mdl.param_slots(), ac);
            for (int k = 0; k < steps; ++k) losses.push_back(train_step(ctx, mdl, opt, sched, local, &led).loss);
        } else {
            parts = pp_forward_backward(ctx, mdl, sched, local, &led);
        }
        std::vector<ParamSlot> slots = mdl.param_slots();
        const std::string path = ep > 1 ? std::string(argv[1]) + ".rank" + std::to_string(ctx.coord().ep) : argv[1];
        FILE* f = std::fopen(path.c_str(), "wb");
        if (!f) {
            rc = 1;
            return;
        }
        std::fprintf(f, "%.17g %.17g %d", parts.ce_sum, parts.aux_sum, (int)slots.size());
        for (double l : losses) std::fprintf(f, " %.17g", l);
        std::fprintf(f, "\n");
        for (const ParamSlot& s : slots) {
            const TensorF* t = steps > 0 ? s.weight : s.grad;
            std::fprintf(f, "%s %lld\n", s.name.c_str(), (long long)t->numel());
            std::fwrite(t->data(), sizeof(float), (size_t)t->numel(), f);
        }
        std::fclose(f);
    });
    return rc;
}
