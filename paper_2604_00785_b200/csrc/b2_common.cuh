// Shared device/host helpers for the B200 MoE expert path and EPSO optimizer.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>
#include <utility>

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

// ---- programmatic dependent launch (PDL) --------------------------------------------
// Every hot-path kernel starts with pdl_wait() (griddepcontrol.wait: the previous kernel on
// the stream has completed and its memory is visible) followed by pdl_launch() (lets the
// next kernel be scheduled now). Kernels launched through launch_k() carry the programmatic
// stream-serialisation attribute, so the next kernel's launch and prologue overlap this
// one's tail; inside CUDA graphs these become programmatic edges. Without the attribute
// both instructions are no-ops.
__device__ __forceinline__ void pdl_wait() {
#if defined(__CUDA_ARCH__) && __CUDA_ARCH__ >= 900
    asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}
__device__ __forceinline__ void pdl_launch() {
#if defined(__CUDA_ARCH__) && __CUDA_ARCH__ >= 900
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}
// programmatic dependent launch (the next kernel's launch and prologue overlap the previous
// one's tail), per host thread (capi.cpp); MoeLayer scopes it per call (see PdlScope)
bool pdl_enabled();
void set_pdl_enabled(bool on);
struct PdlScope {
    bool prev;
    explicit PdlScope(bool on) : prev(pdl_enabled()) { set_pdl_enabled(on); }
    ~PdlScope() { set_pdl_enabled(prev); }
    PdlScope(const PdlScope&) = delete;
    PdlScope& operator=(const PdlScope&) = delete;
};

template <typename... KArgs, typename... Args>
inline void launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    B2_CUDA(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}

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
