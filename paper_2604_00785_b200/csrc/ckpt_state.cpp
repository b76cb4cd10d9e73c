// Shard files of the sharded-optimizer checkpoint over the record-file format:
//   write: write_state_dir's shard part (reference src/reliability.cpp:402-460)
//   read:  restore_full's per-parameter loop (reference src/reliability.cpp:623-675)
// The manifest, the commit marker and the two-slot rotation (CheckpointSet,
// reliability.hpp:120-160) are host bookkeeping around these files and stay with the caller.
#include "ckpt_state.h"

#include <memory>

#include "../../include/b2moe.h"

namespace b2 {

namespace {

// reliability.cpp:322-328 over the rank layout of comm.hpp:45-59
int model_shard_index(const Context& c, int ep_coord) { return (c.coord_pp * c.ep + ep_coord) * c.tp + c.coord_tp; }
int scattered_writer(int model_shard, int dp) { return model_shard % dp; }

std::string shard_file(const std::string& dir, int m) { return dir + "/shard-" + std::to_string(m) + ".bin"; }

std::vector<int64_t> dims_of(const std::vector<std::vector<int64_t>>& dims, int p, int64_t numel) {
    if ((size_t)p < dims.size() && !dims[(size_t)p].empty()) {
        int64_t n = 1;
        for (int64_t d : dims[(size_t)p]) n *= d;
        check(n == numel, "checkpoint: shape of parameter " + std::to_string(p) + " does not cover its elements");
        return dims[(size_t)p];
    }
    return {numel};
}

struct DevBuf {
    float* p = nullptr;
    cudaStream_t st = nullptr;
    DevBuf(int64_t n, cudaStream_t s) : st(s) { B2_CUDA(cudaMallocAsync((void**)&p, 4 * (size_t)std::max<int64_t>(n, 1), s)); }
    ~DevBuf() {
        if (p) cudaFreeAsync(p, st);
    }
};

}  // namespace

ShardWritten write_state_shard(ShardedOptimizer& opt, const std::string& dir, const std::vector<std::string>& names,
                               const std::vector<std::vector<int64_t>>& dims, bool full) {
    Context& c = opt.context();
    const int np = opt.num_params();
    check((int)names.size() == np, "checkpoint: one name per parameter");
    B2_CUDA(cudaSetDevice(c.device));
    ShardWritten out;
    out.model_shard = model_shard_index(c, c.coord_ep);
    out.writer = scattered_writer(out.model_shard, c.dp) == c.coord_dp;
    std::unique_ptr<RecordWriter> w;
    if (out.writer) w = std::make_unique<RecordWriter>(c.device, c.stream, shard_file(dir, out.model_shard));
    for (int i = 0; i < np; ++i) {
        const ParamSlot& p = opt.param(i);
        const bool stores = p.expert || c.coord_ep == 0;
        if (!stores && !(full && opt.over_dp_ep(i))) continue;  // someone else's group assembles this one
        const int64_t n = p.numel;
        std::unique_ptr<DevBuf> ma, m1, m2;
        if (full) {  // slices owned by other replicas are assembled first (reliability.cpp:413-440)
            ma = std::make_unique<DevBuf>(n, c.stream);
            m1 = std::make_unique<DevBuf>(n, c.stream);
            m2 = std::make_unique<DevBuf>(n, c.stream);
            opt.gather_state_device(i, ma->p, m1->p, m2->p);
        }
        if (out.writer && stores) {  // record order of reliability.cpp:448-455
            const std::vector<int64_t> shape = dims_of(dims, i, n);
            w->add(names[(size_t)i] + ".w16", RecDtype::bf16, shape, p.weight, opt.weight_dtype());
            if (full) {
                w->add(names[(size_t)i] + ".master", RecDtype::f32, {n}, ma->p, B2_F32);
                w->add(names[(size_t)i] + ".m", RecDtype::f32, {n}, m1->p, B2_F32);
                w->add(names[(size_t)i] + ".v", RecDtype::f32, {n}, m2->p, B2_F32);
                w->add(names[(size_t)i] + ".g16", RecDtype::bf16, shape, p.grad, opt.grad_dtype());
            }
        }
    }
    if (w) {
        const RecordWriter::Written done = w->finish();
        out.bytes = done.bytes;
        out.crc = done.crc;
    }
    B2_CUDA(cudaStreamSynchronize(c.stream));
    return out;
}

void restore_state_shard(ShardedOptimizer& opt, const std::string& dir, const std::vector<std::string>& names,
                         const std::vector<std::vector<int64_t>>& dims, bool full) {
    Context& c = opt.context();
    const int np = opt.num_params();
    check((int)names.size() == np, "checkpoint: one name per parameter");
    B2_CUDA(cudaSetDevice(c.device));
    const int m = model_shard_index(c, c.coord_ep), m0 = model_shard_index(c, 0);
    std::unique_ptr<RecordFile> fm, fm0;  // each validated once, on first use
    auto file = [&](bool expert) -> RecordFile& {
        std::unique_ptr<RecordFile>& f = (expert || m == m0) ? fm : fm0;
        if (!f) f = std::make_unique<RecordFile>(c.device, c.stream, shard_file(dir, expert ? m : m0));
        return *f;
    };
    auto rec = [&](RecordFile& f, const std::string& name) {
        const int r = f.find(name);
        if (r < 0) throw IoError(dir + ": record '" + name + "' missing");
        return r;
    };
    for (int i = 0; i < np; ++i) {
        const ParamSlot& p = opt.param(i);
        const int64_t n = p.numel;
        const std::vector<int64_t> shape = dims_of(dims, i, n);
        // with the parameter's dims given, the record's shape must match them exactly (restore_full,
        // reliability.cpp:654); without, only its element count is checked
        const bool have_dims = (size_t)i < dims.size() && !dims[(size_t)i].empty();
        auto shape_ok = [&](const RecordInfo& r) { return have_dims ? r.dims == shape : r.numel == n; };
        RecordFile& f = file(p.expert);
        const std::string& nm = names[(size_t)i];
        const int rw = rec(f, nm + ".w16");
        if (!shape_ok(f.records()[(size_t)rw]))
            throw ContractError(dir + ": record '" + nm + ".w16' has the wrong shape");
        f.read(rw, 0, n, p.weight, opt.weight_dtype());
        if (!full) continue;
        int64_t b = 0, e = 0;
        opt.owned(i, &b, &e);
        float *sm = nullptr, *s1 = nullptr, *s2 = nullptr;
        opt.state_slices(i, &sm, &s1, &s2);
        const int ra = rec(f, nm + ".master"), r1 = rec(f, nm + ".m"), r2 = rec(f, nm + ".v");
        for (int r : {ra, r1, r2})
            if (f.records()[(size_t)r].numel != n)
                throw ContractError(dir + ": optimizer records for '" + nm + "' have the wrong size");
        f.read(ra, b, e, sm, B2_F32);
        f.read(r1, b, e, s1, B2_F32);
        f.read(r2, b, e, s2, B2_F32);
        const int rg = rec(f, nm + ".g16");
        if (!shape_ok(f.records()[(size_t)rg]))
            throw ContractError(dir + ": record '" + nm + ".g16' has the wrong shape");
        f.read(rg, 0, n, const_cast<void*>(p.grad), opt.grad_dtype());
    }
}

}  // namespace b2
