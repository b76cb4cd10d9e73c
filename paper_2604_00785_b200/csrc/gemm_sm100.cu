// Grouped expert GEMMs of the SwiGLU FFN on the 5th-generation tensor cores
// (tcgen05 + TMEM + TMA, sm_100a), forward and backward.
//
// Reference: grouped_mm / grouped_mm_nt / grouped_mm_weight_grad
// (include/optimus/kernels.hpp:111-189) as called by expert_forward (moe.hpp:233-236)
// and fast_moe_backward (moe.hpp:406-415), with silu_glu / silu_glu_backward
// (kernels.hpp:262-295) fused into the epilogues and the 1/EP expert-grad scaling
// (moe.hpp:458-461) folded into the weight-gradient store.
//
// One persistent kernel per GEMM kind; per CTA (one per SM, 384 threads):
//   warp 0      TMA producer (one elected lane): A/B tiles -> 4-stage smem ring
//   warp 1      MMA issuer (one lane): tcgen05.mma.cta_group::1.kind::f16,
//               128 x 256 x 16 per instruction, fp32 accumulators in TMEM
//   warp 2      TMEM allocator (512 columns = two 128x256 fp32 accumulators)
//   warps 4-11  epilogue: tcgen05.ld -> registers -> fused math -> global; warp w
//               reads TMEM lanes 32*(w%4).. and half of the tile's columns
// Two accumulators let the epilogue of tile i overlap the MMAs of tile i+1.
//
// Rows of every expert group are padded to 128 in the permuted buffers, so an
// M-tile (forward / dgrad) or a 64-row K-block (wgrad) never straddles experts.
// Operand majors follow the reference layouts with no transposes:
//   FwdGateUp   A = mlp_in [P,H] K-major    B = Wg|Wu [H,I] MN-major (gate||up tile)
//   FwdDown     A = h [P,I] K-major         B = Wd [I,H] MN-major
//   BwdDownDgrad A = dY [P,H] K-major       B = Wd^T: K-major view of [I,H]
//   BwdDx       A = dGU [P,2I] K-major      B = [Wg|Wu]^T: K-major views of [H,I]
//   WgradDown   A = h^T  (MN-major)         B = dY (MN-major), K = rows of the expert
//   WgradGateUp A = X^T  (MN-major)         B = dGU (MN-major)
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstring>
#include <mutex>

#include "b2_common.cuh"
#include "kernels.h"

namespace b2 {
namespace sm100 {

constexpr int BM = 128, BN = 256, BK = 64, STAGES = 4;
constexpr int A_BYTES = BM * BK * 2;           // 16 KB
constexpr int B_BYTES = BN * BK * 2;           // 32 KB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;  // 48 KB
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
constexpr int TMEM_COLS = 512;
constexpr int NUM_EPI_WARPS = 8;  // two warps per TMEM lane quadrant, each half the columns
constexpr int NUM_THREADS = 128 + 32 * NUM_EPI_WARPS;

struct Params {
    CUtensorMap mapA;
    CUtensorMap mapB0;
    CUtensorMap mapB1;
    const int32_t* pad_start;  // [nr+1]
    int nr, H, I;
    int m_tiles_fixed;  // by_k kinds: tiles along M
    int n_tiles;
    int num_kb_fixed;   // by_m kinds: K / BK
    const __nv_bfloat16* g;  // dgrad epilogue inputs
    const __nv_bfloat16* u;
    __nv_bfloat16* out0;
    __nv_bfloat16* out1;
    __nv_bfloat16* out2;
    float scale;
};

// ---------------------------------------------------------------- PTX helpers

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    uint32_t done = 0;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(bar), "r"(parity)
            : "memory");
    } while (!done);
}

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
        "l"((uint64_t)map), "r"(bar), "r"(c0), "r"(c1)
        : "memory");
}
__device__ __forceinline__ void prefetch_map(const CUtensorMap* map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)map) : "memory");
}

// UMMA shared-memory descriptor, SWIZZLE_128B, SM100 version bits
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;  // descriptor version (sm100)
    d |= (uint64_t)2 << 61;  // SWIZZLE_128B
    return d;
}

// kind::f16 instruction descriptor: bf16 x bf16 -> fp32, M = 128, N = 256
__host__ __device__ constexpr uint32_t umma_idesc(bool a_mn, bool b_mn) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16) |
           ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
}

__device__ __forceinline__ void umma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accum) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum)
        : "memory");
}
__device__ __forceinline__ void umma_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
    __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ float bf16_lo(uint32_t v) { return __uint_as_float(v << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t v) { return __uint_as_float(v & 0xFFFF0000u); }

// store 32 fp32 values (scaled) as bf16 to dst[0..32) with column mask `valid`
__device__ __forceinline__ void store_row32(__nv_bfloat16* dst, const float* v, int valid) {
    if (valid >= 32 && ((uintptr_t)dst & 15) == 0) {
        uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
        for (int q = 0; q < 4; ++q)
            d4[q] = make_uint4(pack_bf16(v[8 * q + 0], v[8 * q + 1]), pack_bf16(v[8 * q + 2], v[8 * q + 3]),
                               pack_bf16(v[8 * q + 4], v[8 * q + 5]), pack_bf16(v[8 * q + 6], v[8 * q + 7]));
    } else {
#pragma unroll
        for (int j = 0; j < 32; ++j)
            if (j < valid) dst[j] = __float2bfloat16_rn(v[j]);
    }
}

// ---------------------------------------------------------------- kinds

template <GemmKind K>
struct Traits;
template <>
struct Traits<GemmKind::FwdGateUp> {
    static constexpr bool by_k = false, a_mn = false, b_mn = true;
};
template <>
struct Traits<GemmKind::FwdDown> {
    static constexpr bool by_k = false, a_mn = false, b_mn = true;
};
template <>
struct Traits<GemmKind::BwdDownDgrad> {
    static constexpr bool by_k = false, a_mn = false, b_mn = false;
};
template <>
struct Traits<GemmKind::BwdDx> {
    static constexpr bool by_k = false, a_mn = false, b_mn = false;
};
template <>
struct Traits<GemmKind::WgradDown> {
    static constexpr bool by_k = true, a_mn = true, b_mn = true;
};
template <>
struct Traits<GemmKind::WgradGateUp> {
    static constexpr bool by_k = true, a_mn = true, b_mn = true;
};

struct TileInfo {
    int e;       // expert
    int m0, n0;  // by_m: m0 = padded row; by_k: m0 = output row within the expert
    int kb;      // number of 64-wide K blocks
    int krow0;   // by_k: first padded row of the expert
};

template <GemmKind KIND>
__device__ __forceinline__ int total_tiles(const Params& p, const int32_t* ps) {
    if (Traits<KIND>::by_k) return p.nr * p.m_tiles_fixed * p.n_tiles;
    return (ps[p.nr] / BM) * p.n_tiles;
}

template <GemmKind KIND>
__device__ __forceinline__ TileInfo tile_info(const Params& p, const int32_t* ps, int t) {
    TileInfo ti;
    if (Traits<KIND>::by_k) {
        const int per_e = p.m_tiles_fixed * p.n_tiles;
        ti.e = t / per_e;
        const int r = t % per_e;
        ti.m0 = (r / p.n_tiles) * BM;
        ti.n0 = (r % p.n_tiles) * BN;
        ti.krow0 = ps[ti.e];
        ti.kb = (ps[ti.e + 1] - ps[ti.e]) / BK;
    } else {
        const int mt = t / p.n_tiles;
        ti.n0 = (t % p.n_tiles) * BN;
        ti.m0 = mt * BM;
        int lo = 0, hi = p.nr - 1;  // last expert whose padded start <= m0
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (ps[mid] <= ti.m0) lo = mid;
            else hi = mid - 1;
        }
        ti.e = lo;
        ti.krow0 = 0;
        ti.kb = p.num_kb_fixed;
    }
    return ti;
}

// producer: one stage of A and B for (tile, kb)
template <GemmKind KIND>
__device__ __forceinline__ void load_stage(const Params& p, const TileInfo& ti, int kb, uint32_t sA, uint32_t sB,
                                           uint32_t bar) {
    const int k0 = kb * BK;
    if constexpr (KIND == GemmKind::FwdGateUp) {
        tma_load_2d(sA, &p.mapA, bar, k0, ti.m0);
        const int row = ti.e * p.H + k0;
        const int n0 = ti.n0 / 2;  // 128 gate columns + 128 up columns per tile
        tma_load_2d(sB + 0 * 8192, &p.mapB0, bar, n0, row);
        tma_load_2d(sB + 1 * 8192, &p.mapB0, bar, n0 + 64, row);
        tma_load_2d(sB + 2 * 8192, &p.mapB1, bar, n0, row);
        tma_load_2d(sB + 3 * 8192, &p.mapB1, bar, n0 + 64, row);
    } else if constexpr (KIND == GemmKind::FwdDown) {
        tma_load_2d(sA, &p.mapA, bar, k0, ti.m0);
        const int row = ti.e * p.I + k0;
#pragma unroll
        for (int c = 0; c < 4; ++c) tma_load_2d(sB + c * 8192, &p.mapB0, bar, ti.n0 + 64 * c, row);
    } else if constexpr (KIND == GemmKind::BwdDownDgrad) {
        tma_load_2d(sA, &p.mapA, bar, k0, ti.m0);
        tma_load_2d(sB, &p.mapB0, bar, k0, ti.e * p.I + ti.n0);
    } else if constexpr (KIND == GemmKind::BwdDx) {
        tma_load_2d(sA, &p.mapA, bar, k0, ti.m0);
        if (k0 < p.I) tma_load_2d(sB, &p.mapB0, bar, k0, ti.e * p.H + ti.n0);
        else tma_load_2d(sB, &p.mapB1, bar, k0 - p.I, ti.e * p.H + ti.n0);
    } else {  // wgrad: K runs over the expert's rows; both operands MN-major
        const int row = ti.krow0 + k0;
        tma_load_2d(sA + 0, &p.mapA, bar, ti.m0, row);
        tma_load_2d(sA + 8192, &p.mapA, bar, ti.m0 + 64, row);
#pragma unroll
        for (int c = 0; c < 4; ++c) tma_load_2d(sB + c * 8192, &p.mapB0, bar, ti.n0 + 64 * c, row);
    }
}

__device__ __forceinline__ float silu_f(float x) { return __fdividef(x, 1.f + __expf(-x)); }

// epilogue for one 32-column chunk of one row (thread = row)
template <GemmKind KIND>
__device__ __forceinline__ void epilogue_tile(const Params& p, const TileInfo& ti, uint32_t tacc, int row_in_tile,
                                              bool zero, int half) {
    uint32_t r[32], r2[32];
    float v[32];
    if constexpr (KIND == GemmKind::FwdGateUp) {
        const int64_t row = ti.m0 + row_in_tile;
        const int nbase = ti.n0 / 2;
#pragma unroll 1
        for (int c = half * (BN / 4); c < (half + 1) * (BN / 4); c += 32) {
            tmem_ld32(tacc + c, r);
            tmem_ld32(tacc + BN / 2 + c, r2);
            tmem_wait_ld();
            const int col = nbase + c;
            const int valid = p.I - col;
            if (valid <= 0) continue;
            float gv[32], uv[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                gv[j] = __uint_as_float(r[j]);
                uv[j] = __uint_as_float(r2[j]);
            }
            // G and U are stored rounded to bf16; H is computed from the rounded values
#pragma unroll
            for (int j = 0; j < 32; j += 2) {
                const uint32_t gp = pack_bf16(gv[j], gv[j + 1]), up = pack_bf16(uv[j], uv[j + 1]);
                gv[j] = bf16_lo(gp);
                gv[j + 1] = bf16_hi(gp);
                uv[j] = bf16_lo(up);
                uv[j + 1] = bf16_hi(up);
            }
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = silu_f(gv[j]) * uv[j];
            store_row32(p.out0 + row * p.I + col, gv, valid);
            store_row32(p.out1 + row * p.I + col, uv, valid);
            store_row32(p.out2 + row * p.I + col, v, valid);
        }
    } else if constexpr (KIND == GemmKind::FwdDown || KIND == GemmKind::BwdDx) {
        const int64_t row = ti.m0 + row_in_tile;
#pragma unroll 1
        for (int c = half * (BN / 2); c < (half + 1) * (BN / 2); c += 32) {
            tmem_ld32(tacc + c, r);
            tmem_wait_ld();
            const int col = ti.n0 + c;
            const int valid = p.H - col;
            if (valid <= 0) continue;
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
            store_row32(p.out0 + row * p.H + col, v, valid);
        }
    } else if constexpr (KIND == GemmKind::BwdDownDgrad) {
        // SwiGLU backward (kernels.hpp:277-295): dup = silu(g)*d, dgate = u*d*silu'(g).
        // The G/U loads of a chunk are issued before its TMEM load so they overlap.
        const int64_t row = ti.m0 + row_in_tile;
#pragma unroll 1
        for (int c = half * (BN / 2); c < (half + 1) * (BN / 2); c += 32) {
            const int col = ti.n0 + c;
            const int valid = p.I - col;
            uint4 g4[4], u4[4];
            const __nv_bfloat16* gp = p.g + row * p.I + col;
            const __nv_bfloat16* up = p.u + row * p.I + col;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                g4[q] = make_uint4(0, 0, 0, 0);
                u4[q] = make_uint4(0, 0, 0, 0);
            }
            if (valid >= 32) {
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    g4[q] = __ldg(reinterpret_cast<const uint4*>(gp) + q);
                    u4[q] = __ldg(reinterpret_cast<const uint4*>(up) + q);
                }
            }
            tmem_ld32(tacc + c, r);
            tmem_wait_ld();
            if (valid <= 0) continue;
            float dgv[32], duv[32];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint32_t gw[4] = {g4[q].x, g4[q].y, g4[q].z, g4[q].w};
                const uint32_t uw[4] = {u4[q].x, u4[q].y, u4[q].z, u4[q].w};
#pragma unroll
                for (int h = 0; h < 4; ++h) {
#pragma unroll
                    for (int s = 0; s < 2; ++s) {
                        const int j = 8 * q + 2 * h + s;
                        float x = s ? bf16_hi(gw[h]) : bf16_lo(gw[h]);
                        float uu = s ? bf16_hi(uw[h]) : bf16_lo(uw[h]);
                        if (valid < 32) {
                            x = j < valid ? __bfloat162float(gp[j]) : 0.f;
                            uu = j < valid ? __bfloat162float(up[j]) : 0.f;
                        }
                        const float d = __uint_as_float(r[j]);
                        const float sg = __fdividef(1.f, 1.f + __expf(-x));
                        duv[j] = x * sg * d;
                        dgv[j] = uu * d * (sg * (1.f + x * (1.f - sg)));
                    }
                }
            }
            store_row32(p.out0 + row * 2 * p.I + col, dgv, valid);
            store_row32(p.out0 + row * 2 * p.I + p.I + col, duv, valid);
        }
    } else {  // weight gradients: out[e][m][n] * scale
        // tcgen05.ld is warp-collective: every lane loads, only in-range rows store
        const int m = ti.m0 + row_in_tile;
        const int Mtot = (KIND == GemmKind::WgradDown) ? p.I : p.H;
        const bool row_ok = m < Mtot;
#pragma unroll 1
        for (int c = half * (BN / 2); c < (half + 1) * (BN / 2); c += 32) {
            if (!zero) {
                tmem_ld32(tacc + c, r);
                tmem_wait_ld();
            }
            if (!row_ok) continue;
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = zero ? 0.f : __uint_as_float(r[j]) * p.scale;
            const int col = ti.n0 + c;
            if constexpr (KIND == GemmKind::WgradDown) {
                const int valid = p.H - col;
                if (valid <= 0) continue;
                store_row32(p.out0 + ((int64_t)ti.e * p.I + m) * p.H + col, v, valid);
            } else {
                if (col < p.I) {
                    const int valid = p.I - col;
                    store_row32(p.out0 + ((int64_t)ti.e * p.H + m) * p.I + col, v, valid);
                } else {
                    const int valid = 2 * p.I - col;
                    if (valid <= 0) continue;
                    store_row32(p.out1 + ((int64_t)ti.e * p.H + m) * p.I + (col - p.I), v, valid);
                }
            }
        }
    }
}

template <GemmKind KIND>
__global__ void __launch_bounds__(NUM_THREADS, 1) grouped_gemm_kernel(const __grid_constant__ Params p) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    uint8_t* gbase = smem_raw + (base - raw);
    const uint32_t bar0 = base + STAGES * STAGE_BYTES;
    // barrier layout: full[S], empty[S], tfull[2], tempty[2], then the TMEM address slot
    auto full_bar = [&](int s) { return bar0 + 8u * s; };
    auto empty_bar = [&](int s) { return bar0 + 8u * (STAGES + s); };
    auto tfull_bar = [&](int a) { return bar0 + 8u * (2 * STAGES + a); };
    auto tempty_bar = [&](int a) { return bar0 + 8u * (2 * STAGES + 2 + a); };
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(gbase + STAGES * STAGE_BYTES + 8 * (2 * STAGES + 4));

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (warp == 0 && lane == 0) {
        prefetch_map(&p.mapA);
        prefetch_map(&p.mapB0);
        prefetch_map(&p.mapB1);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(full_bar(s), 1);
            mbar_init(empty_bar(s), 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(tfull_bar(a), 1);
            mbar_init(tempty_bar(a), NUM_EPI_WARPS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(TMEM_COLS)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    const int32_t* ps = p.pad_start;
    const int ntiles = total_tiles<KIND>(p, ps);
    constexpr uint32_t idesc = umma_idesc(Traits<KIND>::a_mn, Traits<KIND>::b_mn);

    if (warp == 0) {
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
                const TileInfo ti = tile_info<KIND>(p, ps, t);
                for (int kb = 0; kb < ti.kb; ++kb) {
                    mbar_wait(empty_bar(stage), phase ^ 1u);
                    const uint32_t sA = base + stage * STAGE_BYTES, sB = sA + A_BYTES;
                    mbar_expect_tx(full_bar(stage), STAGE_BYTES);
                    load_stage<KIND>(p, ti, kb, sA, sB, full_bar(stage));
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1u;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            int it = 0;
            for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
                const TileInfo ti = tile_info<KIND>(p, ps, t);
                const int acc = it & 1;
                const uint32_t acc_phase = (it >> 1) & 1;
                mbar_wait(tempty_bar(acc), acc_phase ^ 1u);
                tc_fence_after();
                const uint32_t tacc = tmem_base + acc * BN;
                for (int kb = 0; kb < ti.kb; ++kb) {
                    mbar_wait(full_bar(stage), phase);
                    tc_fence_after();
                    const uint32_t sA = base + stage * STAGE_BYTES, sB = sA + A_BYTES;
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k) {
                        uint64_t ad, bd;
                        if (Traits<KIND>::a_mn) ad = umma_desc(sA + k * 2048, 8192, 1024);
                        else ad = umma_desc(sA + k * 32, 16, 1024);
                        if (Traits<KIND>::b_mn) bd = umma_desc(sB + k * 2048, 8192, 1024);
                        else bd = umma_desc(sB + k * 32, 16, 1024);
                        umma_f16(tacc, ad, bd, idesc, (kb | k) ? 1u : 0u);
                    }
                    umma_commit(empty_bar(stage));
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1u;
                    }
                }
                if (ti.kb > 0) umma_commit(tfull_bar(acc));
                else mbar_arrive(tfull_bar(acc));
            }
        }
    } else if (warp >= 4) {
        const int quad = warp % 4;        // TMEM lanes 32*quad .. 32*quad+31 (hardware rule: warp id % 4)
        const int half = (warp - 4) / 4;  // column half of the tile
        int it = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
            const TileInfo ti = tile_info<KIND>(p, ps, t);
            const int acc = it & 1;
            const uint32_t acc_phase = (it >> 1) & 1;
            mbar_wait(tfull_bar(acc), acc_phase);
            tc_fence_after();
            const uint32_t tacc = tmem_base + ((uint32_t)(32 * quad) << 16) + acc * BN;
            epilogue_tile<KIND>(p, ti, tacc, 32 * quad + lane, ti.kb == 0, half);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(tempty_bar(acc));
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS)
                     : "memory");
    }
}

// ---------------------------------------------------------------- host side

static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    });
    if (!fn) throw CudaError("cuTensorMapEncodeTiled unavailable");
    return fn;
}

// 2-D bf16 tensor [rows][cols] (cols contiguous), box {bc, br}, 128B swizzle
static CUtensorMap make_map(const void* ptr, int64_t cols, int64_t rows, int bc, int br) {
    CUtensorMap m;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)std::max<int64_t>(rows, 1)};
    cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
    cuuint32_t box[2] = {(cuuint32_t)bc, (cuuint32_t)br};
    cuuint32_t es[2] = {1, 1};
    CUresult r = get_encode()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, es,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
    return m;
}

template <GemmKind KIND>
static void launch_kind(const Params& p, int grid, cudaStream_t st) {
    static std::once_flag once;
    std::call_once(once, [] {
        B2_CUDA(cudaFuncSetAttribute(grouped_gemm_kernel<KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     SMEM_BYTES));
    });
    grouped_gemm_kernel<KIND><<<grid, NUM_THREADS, SMEM_BYTES, st>>>(p);
    B2_LAUNCH_CHECK();
}

}  // namespace sm100

bool sm100_available() {
    int dev = 0, major = 0, minor = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return false;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
    return major == 10 && minor == 0;
}

void launch_sm100_gemm(const Sm100GemmArgs& a, cudaStream_t st) {
    using namespace sm100;
    check(a.H % 64 == 0 && a.I % 64 == 0, "bf16 expert path: hidden and intermediate must be multiples of 64");
    check(a.nr >= 1, "grouped gemm: no local experts");
    if (a.pmax <= 0) return;
    Params p;
    std::memset(&p, 0, sizeof(p));
    p.pad_start = a.pad_start;
    p.nr = a.nr;
    p.H = a.H;
    p.I = a.I;
    p.scale = a.scale;
    p.g = (const __nv_bfloat16*)a.g;
    p.u = (const __nv_bfloat16*)a.u;
    p.out0 = (__nv_bfloat16*)a.out0;
    p.out1 = (__nv_bfloat16*)a.out1;
    p.out2 = (__nv_bfloat16*)a.out2;
    const int64_t P = a.pmax, H = a.H, I = a.I, nr = a.nr;
    int grid = a.num_sms > 0 ? a.num_sms : 148;
    switch (a.kind) {
        case GemmKind::FwdGateUp:
            p.mapA = make_map(a.x, H, P, 64, BM);
            p.mapB0 = make_map(a.wg, I, nr * H, 64, 64);
            p.mapB1 = make_map(a.wu, I, nr * H, 64, 64);
            p.n_tiles = (int)ceil_div(I, BN / 2);
            p.num_kb_fixed = (int)ceil_div(H, BK);
            p.mapB1 = p.mapB1;
            launch_kind<GemmKind::FwdGateUp>(p, grid, st);
            break;
        case GemmKind::FwdDown:
            p.mapA = make_map(a.h, I, P, 64, BM);
            p.mapB0 = make_map(a.wd, H, nr * I, 64, 64);
            p.mapB1 = p.mapB0;
            p.n_tiles = (int)ceil_div(H, BN);
            p.num_kb_fixed = (int)ceil_div(I, BK);
            launch_kind<GemmKind::FwdDown>(p, grid, st);
            break;
        case GemmKind::BwdDownDgrad:
            p.mapA = make_map(a.dy, H, P, 64, BM);
            p.mapB0 = make_map(a.wd, H, nr * I, 64, BN);
            p.mapB1 = p.mapB0;
            p.n_tiles = (int)ceil_div(I, BN);
            p.num_kb_fixed = (int)ceil_div(H, BK);
            launch_kind<GemmKind::BwdDownDgrad>(p, grid, st);
            break;
        case GemmKind::BwdDx:
            p.mapA = make_map(a.dgu, 2 * I, P, 64, BM);
            p.mapB0 = make_map(a.wg, I, nr * H, 64, BN);
            p.mapB1 = make_map(a.wu, I, nr * H, 64, BN);
            p.n_tiles = (int)ceil_div(H, BN);
            p.num_kb_fixed = (int)ceil_div(2 * I, BK);
            launch_kind<GemmKind::BwdDx>(p, grid, st);
            break;
        case GemmKind::WgradDown:
            p.mapA = make_map(a.h, I, P, 64, 64);
            p.mapB0 = make_map(a.dy, H, P, 64, 64);
            p.mapB1 = p.mapB0;
            p.m_tiles_fixed = (int)ceil_div(I, BM);
            p.n_tiles = (int)ceil_div(H, BN);
            grid = (int)std::min<int64_t>(grid, nr * p.m_tiles_fixed * p.n_tiles);
            launch_kind<GemmKind::WgradDown>(p, grid, st);
            break;
        case GemmKind::WgradGateUp:
            p.mapA = make_map(a.x, H, P, 64, 64);
            p.mapB0 = make_map(a.dgu, 2 * I, P, 64, 64);
            p.mapB1 = p.mapB0;
            p.m_tiles_fixed = (int)ceil_div(H, BM);
            p.n_tiles = (int)ceil_div(2 * I, BN);
            grid = (int)std::min<int64_t>(grid, nr * p.m_tiles_fixed * p.n_tiles);
            launch_kind<GemmKind::WgradGateUp>(p, grid, st);
            break;
    }
}

}  // namespace b2
