// Shared device/host helpers for the B200 MoE expert path and EPSO optimizer.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>

namespace b2 {

// Error classes mirror optimus::Error (reference common.hpp:14-36); the C-ABI
// maps them to B2_ERR_* status codes.
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
struct ContractError : Error {
    explicit ContractError(const std::string& m) : Error(1, m) {}
};
struct ConfigError : Error {
    explicit ConfigError(const std::string& m) : Error(2, m) {}
};
struct CudaError : Error {
    explicit CudaError(const std::string& m) : Error(3, m) {}
};

inline void check(bool cond, const std::string& msg) {
    if (!cond) throw ContractError(msg);
}

#define B2_CUDA(call)                                                                    \
    do {                                                                                 \
        cudaError_t e_ = (call);                                                         \
        if (e_ != cudaSuccess)                                                           \
            throw ::b2::CudaError(std::string(#call) + ": " + cudaGetErrorString(e_) +   \
                                  " (" + __FILE__ + ":" + std::to_string(__LINE__) + ")"); \
    } while (0)

#define B2_LAUNCH_CHECK() B2_CUDA(cudaGetLastError())

enum DType : int { F32 = 0, BF16 = 1 };

inline size_t dtype_size(int dt) { return dt == F32 ? 4 : 2; }

// ---- element access, templated on storage type ----------------------------------

template <typename T>
struct Elem;
template <>
struct Elem<float> {
    using Acc = float;      // epilogue / reduction math type
    using Wide = double;    // the reference's fp64 intermediates (silu, softmax)
    __device__ __forceinline__ static float load(const float* p) { return *p; }
    __device__ __forceinline__ static float to_f(float v) { return v; }
    __device__ __forceinline__ static float from_f(float v) { return v; }
};
template <>
struct Elem<__nv_bfloat16> {
    using Acc = float;
    using Wide = float;     // bf16 mode: fp32 math is already below the storage precision
    __device__ __forceinline__ static float load(const __nv_bfloat16* p) { return __bfloat162float(*p); }
    __device__ __forceinline__ static float to_f(__nv_bfloat16 v) { return __bfloat162float(v); }
    __device__ __forceinline__ static __nv_bfloat16 from_f(float v) { return __float2bfloat16_rn(v); }
};

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
__host__ __device__ inline int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }

// rows of each expert group are padded to this multiple inside the permuted
// buffers, so the 256-row GEMM tiles of a CTA pair (forward/dgrad) and the wgrad
// K-blocks never straddle two experts; pad rows are zero and contribute nothing.
constexpr int kRowAlign = 256;

}  // namespace b2
