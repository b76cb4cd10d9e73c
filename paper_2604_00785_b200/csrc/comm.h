// NCCL communicators of one rank, split from the world by the reference's rank
// layout rank = ((pp*DP + dp)*EP + ep)*TP + tp (include/optimus/comm.hpp:45-59), and
// the variable-size collectives the sharded optimizer needs. Member order inside
// every communicator equals the reference's ProcessGroup order (comm.cpp:301-361).
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>
#include <stdint.h>

#include "b2_common.cuh"

namespace b2 {

struct NcclError : Error {
    explicit NcclError(const std::string& m) : Error(4, m) {}
};

#define B2_NCCL(call)                                                                                        \
    do {                                                                                                     \
        ncclResult_t r_ = (call);                                                                            \
        if (r_ != ncclSuccess) throw ::b2::NcclError(std::string(#call) + ": " + ncclGetErrorString(r_)); \
    } while (0)

struct Group {
    ncclComm_t comm = nullptr;
    int size = 1, pos = 0;
};

struct Comm {
    Group world, dp, ep, dp_ep;
    ~Comm();
};

Comm* comm_create(const uint8_t id[128], int rank, int dp, int ep, int tp, int pp, int cdp, int cep, int ctp, int cpp,
                  int device);

ncclDataType_t nccl_dtype(int dtype);

// reducescatterv with the reference's shard_slice bounds (optim.cpp:43-50): member i
// receives the sum of [i*base, i*base+base) (+ the remainder on the last member).
void reduce_scatter_v(const Group& g, const void* src, void* dst, int64_t numel, int dtype, cudaStream_t st);
// allgatherv in place on `buf` (optim.cpp:185-190): member i contributes its slice
void all_gather_v(const Group& g, void* buf, int64_t numel, int dtype, cudaStream_t st);
void all_reduce_sum(const Group& g, const void* src, void* dst, int64_t n, ncclDataType_t dt, cudaStream_t st);

}  // namespace b2
