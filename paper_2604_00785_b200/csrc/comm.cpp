// NCCL plumbing over NVLink/NVSwitch for the EPSO optimizer (see comm.h).
#include "comm.h"

#include <cstring>

namespace b2 {

Comm::~Comm() {
    for (Group* g : {&dp, &ep, &dp_ep})
        if (g->comm && g->comm != world.comm) ncclCommDestroy(g->comm);
    if (world.comm) ncclCommDestroy(world.comm);
}

static Group split(ncclComm_t world, int color, int key, int size) {
    Group g;
    g.size = size;
    g.pos = key;
    if (size == 1) return g;
    B2_NCCL(ncclCommSplit(world, color, key, &g.comm, nullptr));
    return g;
}

Comm* comm_create(const uint8_t id_bytes[128], int rank, int dp, int ep, int tp, int pp, int cdp, int cep, int ctp,
                  int cpp, int device) {
    const int world = dp * ep * tp * pp;
    Comm* c = new Comm();
    try {
        B2_CUDA(cudaSetDevice(device));
        ncclUniqueId id;
        static_assert(sizeof(id) == 128, "ncclUniqueId size");
        std::memcpy(&id, id_bytes, 128);
        B2_NCCL(ncclCommInitRank(&c->world.comm, world, id, rank));
        c->world.size = world;
        c->world.pos = rank;
        // dp group: vary dp with (pp, ep, tp) fixed (comm.cpp:301-311)
        c->dp = split(c->world.comm, (cpp * ep + cep) * tp + ctp, cdp, dp);
        // ep group: vary ep with (pp, dp, tp) fixed (comm.cpp:325-335)
        c->ep = split(c->world.comm, (cpp * dp + cdp) * tp + ctp, cep, ep);
        // fused dp x ep group, dp outer / ep inner (comm.cpp:349-361)
        if (dp * ep == world) {
            c->dp_ep = c->world;  // position (dp*EP + ep)*TP + tp == rank when tp = pp = 1
            c->dp_ep.pos = cdp * ep + cep;
            c->dp_ep.size = dp * ep;
        } else {
            c->dp_ep = split(c->world.comm, cpp * tp + ctp, cdp * ep + cep, dp * ep);
        }
    } catch (...) {
        delete c;
        throw;
    }
    return c;
}

ncclDataType_t nccl_dtype(int dtype) { return dtype == F32 ? ncclFloat32 : ncclBfloat16; }

void reduce_scatter_v(const Group& g, const void* src, void* dst, int64_t numel, int dtype, cudaStream_t st) {
    const size_t es = dtype_size(dtype);
    const int64_t base = numel / g.size, rem = numel - base * g.size;
    const ncclDataType_t dt = nccl_dtype(dtype);
    B2_NCCL(ncclGroupStart());
    if (base > 0) B2_NCCL(ncclReduceScatter(src, dst, (size_t)base, dt, ncclSum, g.comm, st));
    if (rem > 0)
        B2_NCCL(ncclReduce((const char*)src + (size_t)base * g.size * es, (char*)dst + (size_t)base * es, (size_t)rem,
                           dt, ncclSum, g.size - 1, g.comm, st));
    B2_NCCL(ncclGroupEnd());
}

void all_gather_v(const Group& g, void* buf, int64_t numel, int dtype, cudaStream_t st) {
    const size_t es = dtype_size(dtype);
    const int64_t base = numel / g.size, rem = numel - base * g.size;
    const ncclDataType_t dt = nccl_dtype(dtype);
    B2_NCCL(ncclGroupStart());
    if (base > 0)
        B2_NCCL(ncclAllGather((const char*)buf + (size_t)g.pos * base * es, buf, (size_t)base, dt, g.comm, st));
    if (rem > 0) {
        char* tail = (char*)buf + (size_t)base * g.size * es;
        B2_NCCL(ncclBroadcast(tail, tail, (size_t)rem, dt, g.size - 1, g.comm, st));
    }
    B2_NCCL(ncclGroupEnd());
}

void all_reduce_sum(const Group& g, const void* src, void* dst, int64_t n, ncclDataType_t dt, cudaStream_t st) {
    if (g.size == 1) {
        if (src != dst) B2_CUDA(cudaMemcpyAsync(dst, src, (size_t)n * (dt == ncclFloat64 ? 8 : dt == ncclFloat32 ? 4 : 2),
                                                cudaMemcpyDeviceToDevice, st));
        return;
    }
    B2_NCCL(ncclAllReduce(src, dst, (size_t)n, dt, ncclSum, g.comm, st));
}

}  // namespace b2
