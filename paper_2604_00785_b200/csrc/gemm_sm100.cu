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
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "b2_common.cuh"
#include "kernels.h"

namespace b2 {
namespace sm100 {

constexpr int BM = 128, BN = 256, BK = 64;
constexpr int A_BYTES = BM * BK * 2;  // 16 KB: the A rows one CTA holds per stage
// CG = CTAs per MMA (cta_group). CG = 1: 128 x 256 tile per CTA, 4 stages of 48 KB.
// CG = 2: 256 x 256 tile per CTA pair (tcgen05.mma.cta_group::2); each CTA holds its
// 128 A rows and HALF of the B columns, so a stage is 32 KB and 6 stages fit.
template <int CG>
struct Cfg {
    static constexpr int B_COLS = BN / CG;                  // B columns held per CTA
    static constexpr int B_BYTES = B_COLS * BK * 2;
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr int STAGES = CG == 1 ? 4 : 6;
    static constexpr int TILE_M = BM * CG;
};
constexpr int TMEM_COLS = 512;
constexpr int NUM_EPI_WARPS = 8;  // two warps per TMEM lane quadrant, each half the columns
constexpr int NUM_THREADS = 128 + 32 * NUM_EPI_WARPS;
// TMA-store epilogue of the six expert kinds: each epilogue warp owns SLOTS 2 KB staging
// slots, each one 32-row x 32-column bf16 box in the SWIZZLE_64B layout
constexpr int EPI_SLOT_BYTES = 32 * 32 * 2;
// Wide tiles: 256 x 512 per CTA pair — two N = 256 MMAs per k-step into one 512-column TMEM
// accumulator. Per SM a k-block then brings 16 KB of A and 32 KB of B for 128 x 512 x 64 MACs
// instead of 16 + 16 KB for 128 x 256 x 64: a quarter fewer L2 -> SM bytes per FLOP, the limit of
// the 256-wide kernels (with the operand loads removed the same MMAs run at the measured bf16
// peak: tools/gemm_tile_probe.py, noload experiment). No accumulator double-buffering is left, so
// the epilogue frees the two 256-column halves separately and the next tile's MMAs start on the
// first half while the second drains.
// Measured per kind at config B (tools/gemm_tile_probe.py, same box): FwdGateUp 837 -> 803 us,
// FwdDown 424 -> 397, BwdDx 819 -> 751, WgradDown 417 -> 394, WgradGateUp 806 -> 756; the dgrad,
// whose epilogue also loads G/U and computes the SwiGLU backward, got slower without the
// double-buffered accumulator (503 -> 562 us) and stays 256 wide.
template <GemmKind K>
struct WideKind {
    static constexpr bool value = K == GemmKind::FwdGateUp || K == GemmKind::FwdDown || K == GemmKind::BwdDx ||
                                  K == GemmKind::WgradDown || K == GemmKind::WgradGateUp;
};
// (the dgrad was also measured wide as four N = 128 regions released one by one, its epilogue
// holding 64 accumulator columns per warp: 475 -> 597 us)
constexpr int MAX_REGIONS = 2;
template <GemmKind K, int CG>
struct KCfg {
    static constexpr bool WIDE = CG == 2 && WideKind<K>::value;
    static constexpr int TN = WIDE ? 2 * BN : BN;  // N columns of a tile
    static constexpr int REGIONS = TN / BN;        // N = 256 MMAs per k-step (accumulator regions)
    static_assert(REGIONS <= MAX_REGIONS, "too many accumulator regions");
    static constexpr int B_COLS = TN / CG;         // B columns held per CTA
    static constexpr int REGION_BYTES = (B_COLS / REGIONS) * BK * 2;
    static constexpr int STAGE_BYTES = A_BYTES + B_COLS * BK * 2;
    static constexpr bool TMA_EPI = (int)K <= (int)GemmKind::WgradGateUp;
    // two staging slots everywhere (FwdGateUp's three boxes per chunk rotate through them)
    static constexpr int SLOTS = 2;
    static constexpr int STAGES = CG == 1 ? 4 : (WIDE ? 4 : 6);
    static constexpr int WARP_EPI_BYTES = TMA_EPI ? SLOTS * EPI_SLOT_BYTES : 0;
    static constexpr int SMEM =
        STAGES * STAGE_BYTES + 1024 /*align*/ + 1024 /*barriers*/ + NUM_EPI_WARPS * WARP_EPI_BYTES;
    static_assert(SMEM <= 232448, "kernel exceeds 227 KB of shared memory");
};

struct Params {
    CUtensorMap mapA;
    CUtensorMap mapA1;  // RouterDx: the low bf16 half of dlogits (K blocks past num_kb_fixed / 2)
    CUtensorMap mapB0;
    CUtensorMap mapB1;
    CUtensorMap mapO0;  // TMA-store maps of the outputs (32 x 32 [x 1] boxes, SWIZZLE_64B)
    CUtensorMap mapO1;
    CUtensorMap mapO2;
    const int32_t* pad_start;  // [nr+1]
    const int32_t* counts;     // [nr] rows per expert (wgrad K extent)
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
    const float* row_w;   // FwdGateUp / BwdDownDgrad: per padded row routing weight (weighted-H scheme)
    float* wpart;         // BwdDownDgrad with row_w: [P, I / 64] partial weight-gradient dots
    const int32_t* eorder;  // by_k kinds: expert of the i-th group of tiles (null: i), longest first
    uint32_t idesc;       // instruction descriptor (runtime N for the router kinds)
    int umma_n;           // accumulator columns in use
    int b_chunks;         // 64-column B boxes per stage (MN-major B)
    uint32_t stage_tx;    // bytes a stage's TMA loads deliver
    int S, N;             // router kinds: tokens, experts
    int rows_per_split;   // RouterDw
    const __nv_bfloat16* src;  // RouterDx: rows added to the router term (the token's summed expert rows)
    float* part;
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
__device__ __forceinline__ uint64_t global_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// bounded spin: a barrier that never completes (a protocol bug) traps after ~20 s instead
// of hanging the GPU; `tag` identifies the waiter in the message
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity, int tag = 0) {
    uint32_t done = 0;
    uint32_t spins = 0;
    uint64_t t0 = 0;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(bar), "r"(parity)
            : "memory");
        if (!done && (++spins & 0xFFFFu) == 0) {
            const uint64_t now = global_ns();
            if (t0 == 0) {
                t0 = now;
            } else if (now - t0 > 20000000000ull) {
                printf("b2 gemm: mbarrier wait stuck (tag %d, block %d, thread %d, parity %u)\n", tag,
                       (int)blockIdx.x, (int)threadIdx.x, parity);
                __trap();
            }
        }
    } while (!done);
}

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
        "l"((uint64_t)map), "r"(bar), "r"(c0), "r"(c1)
        : "memory");
}
// 2-CTA (cta_group::2) load: the bytes complete_tx on the LEADER CTA's barrier
__device__ __forceinline__ void tma_load_2d_cg2(uint32_t dst, const CUtensorMap* map, uint32_t leader_bar, int c0,
                                                int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
        "l"((uint64_t)map), "r"(leader_bar), "r"(c0), "r"(c1)
        : "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
// shared::cluster address of the same smem offset in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t map_to_rank(uint32_t addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
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

// kind::f16 instruction descriptor: bf16 x bf16 -> fp32, M = 128, N = n (16..256, %16)
__host__ __device__ constexpr uint32_t umma_idesc(bool a_mn, bool b_mn, int n = BN, int m = BM) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16) |
           ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
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
__device__ __forceinline__ void umma_f16_cg2(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                             uint32_t accum) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum)
        : "memory");
}
__device__ __forceinline__ void umma_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
// arrive on the same barrier offset in both CTAs of the pair once the MMAs retire
__device__ __forceinline__ void umma_commit_cg2(uint32_t bar) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(bar),
        "h"((uint16_t)0x3)
        : "memory");
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

__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, uint32_t src, int c0, int c1) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"((uint64_t)map),
                 "r"(src), "r"(c0), "r"(c1)
                 : "memory");
}
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, uint32_t src, int c0, int c1, int c2) {
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                     (uint64_t)map),
                 "r"(src), "r"(c0), "r"(c1), "r"(c2)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

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

// Per-warp TMA-store staging. Lane r writes row r of a 32 x 32 bf16 box with four 128-bit
// shared stores (conflict-free under the 64-byte swizzle: unit q of row r lands at unit
// q ^ ((r >> 1) & 3)); lane 0 hands the box to the TMA engine as one bulk group. A slot is
// rewritten only after the engine has read it (wait_group.read of the SLOTS-1 newest groups).
template <int SLOTS>
struct EpiStage {
    uint32_t s0;  // shared address of slot 0
    uint8_t* g0;  // generic address of slot 0
    int slot;
    __device__ __forceinline__ uint32_t begin(int lane, const float* v) {
        uint32_t pk[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) pk[j] = pack_bf16(v[2 * j], v[2 * j + 1]);
        return begin_packed(lane, pk);
    }
    // pk: the row's 32 bf16 values packed in pairs
    __device__ __forceinline__ uint32_t begin_packed(int lane, const uint32_t* pk) {
        if (lane == 0) bulk_wait_read<SLOTS - 1>();
        __syncwarp();
        uint4* row = reinterpret_cast<uint4*>(g0 + slot * EPI_SLOT_BYTES + lane * 64);
        const int sw = (lane >> 1) & 3;
#pragma unroll
        for (int q = 0; q < 4; ++q) row[q ^ sw] = make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
        fence_async_smem();
        __syncwarp();
        const uint32_t src = s0 + slot * EPI_SLOT_BYTES;
        slot = slot + 1 == SLOTS ? 0 : slot + 1;
        return src;
    }
    __device__ __forceinline__ void put2d(const CUtensorMap* map, int lane, const float* v, int c0, int c1) {
        const uint32_t src = begin(lane, v);
        if (lane == 0) {
            tma_store_2d(map, src, c0, c1);
            bulk_commit();
        }
    }
    __device__ __forceinline__ void put2d_packed(const CUtensorMap* map, int lane, const uint32_t* pk, int c0, int c1) {
        const uint32_t src = begin_packed(lane, pk);
        if (lane == 0) {
            tma_store_2d(map, src, c0, c1);
            bulk_commit();
        }
    }
    __device__ __forceinline__ void put3d_packed(const CUtensorMap* map, int lane, const uint32_t* pk, int c0, int c1,
                                                 int c2) {
        const uint32_t src = begin_packed(lane, pk);
        if (lane == 0) {
            tma_store_3d(map, src, c0, c1, c2);
            bulk_commit();
        }
    }
    __device__ __forceinline__ void put3d(const CUtensorMap* map, int lane, const float* v, int c0, int c1, int c2) {
        const uint32_t src = begin(lane, v);
        if (lane == 0) {
            tma_store_3d(map, src, c0, c1, c2);
            bulk_commit();
        }
    }
    __device__ __forceinline__ void drain(int lane) {
        if (lane == 0) bulk_wait_all();
        __syncwarp();
    }
};

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
template <>
struct Traits<GemmKind::RouterDx> {
    static constexpr bool by_k = false, a_mn = false, b_mn = false;
};
template <>
struct Traits<GemmKind::RouterDw> {
    static constexpr bool by_k = true, a_mn = true, b_mn = true;
};

struct TileInfo {
    int e;       // expert
    int m0, n0;  // by_m: m0 = padded row; by_k: m0 = output row within the expert
    int kb;      // number of 64-wide K blocks
    int krow0;   // by_k: first padded row of the expert
};

template <GemmKind KIND, int CG>
__device__ __forceinline__ int total_tiles(const Params& p, const int32_t* ps) {
    if (KIND == GemmKind::RouterDx) return (int)ceil_div(p.S, BM) * p.n_tiles;
    if (Traits<KIND>::by_k) return p.nr * p.m_tiles_fixed * p.n_tiles;
    return (ps[p.nr] / Cfg<CG>::TILE_M) * p.n_tiles;
}

template <GemmKind KIND, int CG>
__device__ __forceinline__ TileInfo tile_info(const Params& p, const int32_t* ps, int t) {
    constexpr int TM = Cfg<CG>::TILE_M;
    TileInfo ti;
    if (KIND == GemmKind::RouterDx) {
        ti.m0 = (t / p.n_tiles) * BM;
        ti.n0 = (t % p.n_tiles) * BN;
        ti.e = 0;
        ti.krow0 = 0;
        ti.kb = p.num_kb_fixed;
        return ti;
    }
    if (KIND == GemmKind::RouterDw) {  // "experts" are the S splits; n_tiles == 1
        ti.e = t / p.m_tiles_fixed;
        ti.m0 = (t % p.m_tiles_fixed) * BM;
        ti.n0 = 0;
        ti.krow0 = ti.e * p.rows_per_split;
        const int rows = min(p.S, ti.krow0 + p.rows_per_split) - ti.krow0;
        ti.kb = rows > 0 ? (rows + BK - 1) / BK : 0;
        return ti;
    }
    if (Traits<KIND>::by_k) {
        const int per_e = p.m_tiles_fixed * p.n_tiles;
        ti.e = p.eorder ? p.eorder[t / per_e] : t / per_e;
        const int r = t % per_e;
        ti.m0 = (r / p.n_tiles) * TM;
        ti.n0 = (r % p.n_tiles) * KCfg<KIND, CG>::TN;
        ti.krow0 = ps[ti.e];
        ti.kb = (p.counts[ti.e] + BK - 1) / BK;  // pad rows past the count are zero: skip them
    } else {
        const int mt = t / p.n_tiles;
        ti.n0 = (t % p.n_tiles) * KCfg<KIND, CG>::TN;
        ti.m0 = mt * TM;
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

// producer: one stage of A and B for (tile, kb). `m_own` is the first A row this CTA
// holds (the pair's tile base + 128 * rank); with CG = 2 each CTA loads B columns
// [128 * rank, 128 * rank + 128) of the tile and signals the leader's barrier.
template <GemmKind KIND, int CG>
__device__ __forceinline__ void load_stage(const Params& p, const TileInfo& ti, int kb, int m_own, uint32_t rank,
                                           uint32_t sA, uint32_t sB, uint32_t bar) {
    const int k0 = kb * BK;
    auto ld = [&](uint32_t dst, const CUtensorMap* map, int c0, int c1) {
        if constexpr (CG == 1) tma_load_2d(dst, map, bar, c0, c1);
        else tma_load_2d_cg2(dst, map, bar, c0, c1);
    };
    // A of the by-row kinds: [m_own, m_own + 128) x [k0, k0 + 64), K-major
    auto ldA_rows = [&]() { ld(sA, &p.mapA, k0, m_own); };
    constexpr int BC = KCfg<KIND, CG>::B_COLS;
    const int nb = ti.n0 + BC * (int)rank;  // this CTA's first B column of the tile (one region)
    if constexpr (KIND == GemmKind::FwdGateUp) {
        ldA_rows();
        const int row = ti.e * p.H + k0;
        // region q: [gate 128 | up 128] columns of I columns n0/2 + 128 q ..; CTA 0 loads the gate
        // half of every region, CTA 1 the up half
        static_assert(CG == 2, "FwdGateUp runs on CTA pairs");
#pragma unroll
        for (int q = 0; q < KCfg<KIND, CG>::REGIONS; ++q) {
            const int n0 = ti.n0 / 2 + (BN / 2) * q;
            const uint32_t d = sB + q * KCfg<KIND, CG>::REGION_BYTES;
            const CUtensorMap* m = rank == 0 ? &p.mapB0 : &p.mapB1;
            ld(d, m, n0, row);
            ld(d + 8192, m, n0 + 64, row);
        }
    } else if constexpr (KIND == GemmKind::FwdDown) {
        ldA_rows();
        const int row = ti.e * p.I + k0;
        // region q (MMA q) holds tile columns 256 q + 128 rank .. of this CTA, 2 boxes of 64
#pragma unroll
        for (int c = 0; c < BC / 64; ++c)
            ld(sB + c * 8192, &p.mapB0, ti.n0 + BN * (c / 2) + (BN / 2) * (int)rank + 64 * (c % 2), row);
    } else if constexpr (KIND == GemmKind::BwdDownDgrad) {
        ldA_rows();
#pragma unroll
        for (int q = 0; q < KCfg<KIND, CG>::REGIONS; ++q)
            ld(sB + q * KCfg<KIND, CG>::REGION_BYTES, &p.mapB0, k0,
               ti.e * p.I + ti.n0 + BN * q + (BN / 2) * (int)rank);
    } else if constexpr (KIND == GemmKind::BwdDx) {
        ldA_rows();
#pragma unroll
        for (int q = 0; q < KCfg<KIND, CG>::REGIONS; ++q) {  // region q: tile rows 256 q + 128 rank ..
            const int r = ti.e * p.H + ti.n0 + BN * q + (BN / 2) * (int)rank;
            const uint32_t d = sB + q * KCfg<KIND, CG>::REGION_BYTES;
            if (k0 < p.I) ld(d, &p.mapB0, k0, r);
            else ld(d, &p.mapB1, k0 - p.I, r);
        }
    } else if constexpr (KIND == GemmKind::RouterDx) {
        // K runs twice over the experts: dl_hi · Wrᵀ, then dl_lo · Wrᵀ into the same accumulator
        const int kh = (p.num_kb_fixed / 2) * BK;
        if (k0 < kh) ld(sA, &p.mapA, k0, ti.m0);
        else ld(sA, &p.mapA1, k0 - kh, ti.m0);
        ld(sB, &p.mapB0, k0 < kh ? k0 : k0 - kh, ti.n0);
    } else if constexpr (KIND == GemmKind::RouterDw) {
        const int row = ti.krow0 + k0;
        ld(sA + 0, &p.mapA, ti.m0, row);
        ld(sA + 8192, &p.mapA, ti.m0 + 64, row);
        for (int c = 0; c < p.b_chunks; ++c) ld(sB + c * 8192, &p.mapB0, 64 * c, row);
    } else {  // wgrad: K runs over the expert's rows; both operands MN-major
        const int row = ti.krow0 + k0;
        ld(sA + 0, &p.mapA, m_own, row);
        ld(sA + 8192, &p.mapA, m_own + 64, row);
#pragma unroll
        for (int c = 0; c < BC / 64; ++c)
            ld(sB + c * 8192, &p.mapB0, ti.n0 + BN * (c / 2) + (BN / 2) * (int)rank + 64 * (c % 2), row);
    }
}

__device__ __forceinline__ float silu_f(float x) { return __fdividef(x, 1.f + __expf(-x)); }

// dgrad epilogue operands: 32 bf16 columns of one row of G and of U (64 B each)
// (32-byte loads: one full sector per request, half the requests of 16-byte ones; dgrad eager
// stage 0.58-0.61 -> 0.58-0.59 ms, three alternated rounds)
__device__ __forceinline__ void ld_nc_256(const void* p, uint4& a, uint4& b) {
    asm volatile("ld.global.nc.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w)
                 : "l"(p));
}
__device__ __forceinline__ void load_gu(const Params& p, int64_t off, uint4 (&g4)[4], uint4 (&u4)[4]) {
    const uint4* gp = reinterpret_cast<const uint4*>(p.g + off);
    const uint4* up = reinterpret_cast<const uint4*>(p.u + off);
#pragma unroll
    for (int q = 0; q < 4; q += 2) {
        ld_nc_256(gp + q, g4[q], g4[q + 1]);
        ld_nc_256(up + q, u4[q], u4[q + 1]);
    }
}

// epilogue of the router kinds for one row (thread = row); the six expert kinds store
// through the TMA-store staging in the kernel body
template <GemmKind KIND>
__device__ __forceinline__ void epilogue_tile(const Params& p, const TileInfo& ti, uint32_t tacc, int row_in_tile,
                                              bool zero, int half) {
    uint32_t r[32];
    float v[32];
    if constexpr (KIND == GemmKind::RouterDx) {
        // dx[t] = base[t] (the token's summed expert rows) + router term (moe.hpp:418-427
        // scatter-add + 454 matmul_nt); rows beyond S only drain TMEM
        const int t = ti.m0 + row_in_tile;
        const bool row_ok = t < p.S;
#pragma unroll 1
        for (int c = half * (BN / 2); c < (half + 1) * (BN / 2); c += 32) {
            tmem_ld32(tacc + c, r);
            tmem_wait_ld();
            const int col = ti.n0 + c;
            const int valid = p.H - col;
            if (!row_ok || valid <= 0) continue;
            float base[32];
            const __nv_bfloat16* sp = p.src + (int64_t)t * p.H + col;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint4 w4 = __ldg(reinterpret_cast<const uint4*>(sp) + q);
                const uint32_t w[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
                for (int h = 0; h < 4; ++h) {
                    base[8 * q + 2 * h] = bf16_lo(w[h]);
                    base[8 * q + 2 * h + 1] = bf16_hi(w[h]);
                }
            }
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = base[j] + __uint_as_float(r[j]);
            store_row32(p.out0 + (int64_t)t * p.H + col, v, valid);
        }
    } else if constexpr (KIND == GemmKind::RouterDw) {
        // fp32 partial of dWr for this S split; half 0 covers all umma_n columns
        if (half != 0) return;
        const int h = ti.m0 + row_in_tile;
        const bool row_ok = h < p.H;
#pragma unroll 1
        for (int c = 0; c < p.umma_n; c += 32) {
            if (!zero) {
                tmem_ld32(tacc + c, r);
                tmem_wait_ld();
            }
            if (!row_ok) continue;
            float* dst = p.part + ((int64_t)ti.e * p.H + h) * p.N + c;
            const int valid = min(32, p.N - c);
            if (valid <= 0) continue;
            if (valid == 32 && (p.N % 4) == 0) {
#pragma unroll
                for (int q = 0; q < 8; ++q)
                    reinterpret_cast<float4*>(dst)[q] =
                        zero ? make_float4(0.f, 0.f, 0.f, 0.f)
                             : make_float4(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]),
                                           __uint_as_float(r[4 * q + 2]), __uint_as_float(r[4 * q + 3]));
            } else {
#pragma unroll
                for (int j = 0; j < 32; ++j)
                    if (j < valid) dst[j] = zero ? 0.f : __uint_as_float(r[j]);
            }
        }
    }
}

template <GemmKind KIND, int CG>
__global__ void __launch_bounds__(NUM_THREADS, 1) grouped_gemm_kernel(const __grid_constant__ Params p) {
    using C = Cfg<CG>;
    using KC = KCfg<KIND, CG>;
    constexpr int STAGES = KC::STAGES;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    uint8_t* gbase = smem_raw + (base - raw);
    const uint32_t bar0 = base + STAGES * KC::STAGE_BYTES;
    // barrier layout: full[S], empty[S], tfull[2], tempty[2], then the TMEM address slot
    auto full_bar = [&](int s) { return bar0 + 8u * s; };
    auto empty_bar = [&](int s) { return bar0 + 8u * (STAGES + s); };
    auto tfull_bar = [&](int a) { return bar0 + 8u * (2 * STAGES + a); };
    auto tempty_bar = [&](int a) { return bar0 + 8u * (2 * STAGES + 2 + a); };
    uint32_t* tmem_slot =
        reinterpret_cast<uint32_t*>(gbase + STAGES * KC::STAGE_BYTES + 8 * (2 * STAGES + 2 + MAX_REGIONS));
    // per epilogue warp: SLOTS output staging boxes; 1 KB aligned (bar0 is)
    const uint32_t epi_base = bar0 + 1024u;

    pdl_launch();  // the next kernel may be scheduled (it waits for this grid's completion)
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    // CG = 2: the cluster is one CTA pair; the leader (rank 0) issues the pair's MMAs
    const uint32_t rank = CG == 2 ? cluster_rank() : 0u;
    const bool leader = rank == 0;
    if (warp == 0 && lane == 0) {
        prefetch_map(&p.mapA);
        prefetch_map(&p.mapB0);
        prefetch_map(&p.mapB1);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(full_bar(s), 1);
            mbar_init(empty_bar(s), 1);
        }
        for (int a = 0; a < 2; ++a) mbar_init(tfull_bar(a), 1);
        for (int a = 0; a < MAX_REGIONS; ++a)
            mbar_init(tempty_bar(a), NUM_EPI_WARPS * CG);  // the leader's counts both CTAs' epilogues
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (warp == 2) {
        if constexpr (CG == 1) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                         "r"(TMEM_COLS)
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
        } else {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                         "r"(TMEM_COLS)
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
        }
    }
    tc_fence_before();
    if constexpr (CG == 2) cluster_sync_all();  // peer barriers initialised before any remote arrive
    else __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    // PDL: the set-up above overlapped the previous kernel's tail; no global memory was
    // touched yet. From here on the previous kernel's results are needed.
    pdl_wait();

    const int32_t* ps = p.pad_start;
    const int ntiles = total_tiles<KIND, CG>(p, ps);
    const uint32_t idesc = p.idesc;
    // persistent tile scheduler: pair (cluster) u takes tiles u, u + npairs, ...
    const int tfirst = blockIdx.x / CG, tstride = gridDim.x / CG;

    if (warp == 0) {
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int t = tfirst; t < ntiles; t += tstride) {
                const TileInfo ti = tile_info<KIND, CG>(p, ps, t);
                const int m_own = ti.m0 + BM * (int)rank;
                for (int kb = 0; kb < ti.kb; ++kb) {
                    mbar_wait(empty_bar(stage), phase ^ 1u, 0);
                    const uint32_t sA = base + stage * KC::STAGE_BYTES, sB = sA + A_BYTES;
                    uint32_t fb = full_bar(stage);
                    if constexpr (CG == 2) fb = map_to_rank(fb, 0);
                    if (leader) mbar_expect_tx(full_bar(stage), p.stage_tx);
                    load_stage<KIND, CG>(p, ti, kb, m_own, rank, sA, sB, fb);
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1u;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0 && leader) {
            int stage = 0;
            uint32_t phase = 0;
            int it = 0;
            for (int t = tfirst; t < ntiles; t += tstride, ++it) {
                const TileInfo ti = tile_info<KIND, CG>(p, ps, t);
                // two double-buffered 256-column accumulators, or (wide) one 512-column accumulator
                // whose halves are freed separately (tempty[0], tempty[1])
                const int acc = KC::WIDE ? 0 : it & 1;
                const uint32_t acc_phase = KC::WIDE ? it & 1 : (it >> 1) & 1;
                if (!KC::WIDE || ti.kb == 0) {
                    mbar_wait(tempty_bar(acc), acc_phase ^ 1u, 2);
                    if (KC::WIDE)
                        for (int q = 1; q < KC::REGIONS; ++q) mbar_wait(tempty_bar(q), acc_phase ^ 1u, 2);
                    tc_fence_after();
                }
                const uint32_t tacc = tmem_base + acc * BN;
                // MMAs of k-block kb into region q (N = 256 columns each)
                auto issue = [&](int stg, int kb, int q) {
                    const uint32_t sA = base + stg * KC::STAGE_BYTES, sB = sA + A_BYTES + q * KC::REGION_BYTES;
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k) {
                        uint64_t ad, bd;
                        if (Traits<KIND>::a_mn) ad = umma_desc(sA + k * 2048, 8192, 1024);
                        else ad = umma_desc(sA + k * 32, 16, 1024);
                        if (Traits<KIND>::b_mn) bd = umma_desc(sB + k * 2048, 8192, 1024);
                        else bd = umma_desc(sB + k * 32, 16, 1024);
                        if constexpr (CG == 1) umma_f16(tacc + q * BN, ad, bd, idesc, (kb | k) ? 1u : 0u);
                        else umma_f16_cg2(tacc + q * BN, ad, bd, idesc, (kb | k) ? 1u : 0u);
                    }
                };
                auto release_stage = [&]() {
                    if constexpr (CG == 1) umma_commit(empty_bar(stage));
                    else umma_commit_cg2(empty_bar(stage));
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1u;
                    }
                };
                int kb0 = 0;
                if constexpr (KC::WIDE) {
                    // the first k-blocks' region-0 MMAs (every loaded stage) run while the epilogue
                    // still drains the later regions of the previous tile; each later region's MMAs
                    // follow as soon as it is released
                    const int na = ti.kb < STAGES ? ti.kb : STAGES;
#pragma unroll 1
                    for (int q = 0; q < KC::REGIONS && na > 0; ++q) {
                        mbar_wait(tempty_bar(q), acc_phase ^ 1u, 2);
                        tc_fence_after();
                        int sj = stage;
                        uint32_t pj = phase;
                        for (int j = 0; j < na; ++j) {
                            if (q == 0) {
                                mbar_wait(full_bar(sj), pj, 1);
                                tc_fence_after();
                            }
                            issue(sj, j, q);
                            if (++sj == STAGES) {
                                sj = 0;
                                pj ^= 1u;
                            }
                        }
                    }
                    for (int j = 0; j < na; ++j) release_stage();
                    kb0 = na;
                }
                for (int kb = kb0; kb < ti.kb; ++kb) {
                    mbar_wait(full_bar(stage), phase, 1);
                    tc_fence_after();
#pragma unroll
                    for (int q = 0; q < KC::REGIONS; ++q) issue(stage, kb, q);
                    release_stage();
                }
                if (ti.kb > 0) {
                    if constexpr (CG == 1) umma_commit(tfull_bar(acc));
                    else umma_commit_cg2(tfull_bar(acc));
                } else {  // empty K range: nothing to wait for, the epilogues store zeros
                    mbar_arrive(tfull_bar(acc));
                    if constexpr (CG == 2) mbar_arrive_cluster(map_to_rank(tfull_bar(acc), 1));
                }
            }
        }
    } else if (warp >= 4) {
        const int quad = warp % 4;        // TMEM lanes 32*quad .. 32*quad+31 (hardware rule: warp id % 4)
        const int half = (warp - 4) / 4;  // column half of the tile
        const uint32_t tempty0 = CG == 2 ? map_to_rank(tempty_bar(0), 0) : tempty_bar(0);
        const int ew = warp - 4;
        EpiStage<KC::SLOTS> stg;
        stg.s0 = epi_base + (uint32_t)(ew * KC::WARP_EPI_BYTES);
        stg.g0 = gbase + (stg.s0 - base);
        stg.slot = 0;
        const int row0 = 32 * quad;  // first row of this warp inside the CTA's 128
        int it = 0;
        for (int t = tfirst; t < ntiles; t += tstride, ++it) {
            TileInfo ti = tile_info<KIND, CG>(p, ps, t);
            ti.m0 += BM * (int)rank;  // this CTA's 128 rows of the pair's tile
            const int acc = KC::WIDE ? 0 : it & 1;
            const uint32_t acc_phase = KC::WIDE ? it & 1 : (it >> 1) & 1;
            // this lane's row weight and (dgrad) G/U operands of the first chunk load while the
            // MMAs still run
            float wrow = 1.f;
            if constexpr (KIND == GemmKind::FwdGateUp || KIND == GemmKind::BwdDownDgrad)
                if (p.row_w) wrow = __ldg(p.row_w + ti.m0 + row0 + lane);
            uint4 gq[4], uq[4];
            if constexpr (KIND == GemmKind::BwdDownDgrad) {
                const int col = ti.n0 + half * (BN / 2);
                if (col < p.I) load_gu(p, (int64_t)(ti.m0 + row0 + lane) * p.I + col, gq, uq);
            }
            mbar_wait(tfull_bar(acc), acc_phase, 3);
            tc_fence_after();
            const uint32_t tacc0 = tmem_base + ((uint32_t)(32 * quad) << 16) + acc * BN;
            // drain one 256-column accumulator (`tacc`) holding tile columns ti.n0 ..
            auto drain = [&](const uint32_t tacc, const TileInfo& ti) {
                if constexpr (KIND == GemmKind::BwdDownDgrad) {
                    // SwiGLU backward (kernels.hpp:277-295) on the dH accumulator. G and U of this lane's
                    // row come straight from global into registers (ld.global.nc), one 32-column chunk
                    // ahead of the math (the first one before the accumulator wait). Weighted-H scheme
                    // (row_w): the accumulator is dH' = dout . Wd^T; dmul = w * dH', and the row's
                    // top-k weight-gradient partial dH' . silu(G) * U (= dout . y) goes to wpart
                    const bool wscheme = p.row_w != nullptr;
                    const int64_t grow = (int64_t)(ti.m0 + row0 + lane) * p.I;
                    float wdot = 0.f;
    #pragma unroll 1
                    for (int c = half * (BN / 2); c < (half + 1) * (BN / 2); c += 32) {
                        const int col = ti.n0 + c;
                        const bool live = col < p.I;  // I % 64 == 0: a chunk is all in or all out
                        uint4 g4[4], u4[4];
    #pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            g4[q] = gq[q];
                            u4[q] = uq[q];
                        }
                        if (c + 32 < (half + 1) * (BN / 2) && col + 32 < p.I) load_gu(p, grow + col + 32, gq, uq);
                        uint32_t r[32];
                        tmem_ld32(tacc + c, r);
                        tmem_wait_ld();
                        if (!live) continue;
                        uint32_t dgp[16], dup[16];
    #pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            const uint32_t gw[4] = {g4[q].x, g4[q].y, g4[q].z, g4[q].w},
                                           uw[4] = {u4[q].x, u4[q].y, u4[q].z, u4[q].w};
    #pragma unroll
                            for (int h = 0; h < 4; ++h) {
                                float dg2[2], du2[2];
    #pragma unroll
                                for (int e = 0; e < 2; ++e) {
                                    const float x = e ? bf16_hi(gw[h]) : bf16_lo(gw[h]);
                                    const float uu = e ? bf16_hi(uw[h]) : bf16_lo(uw[h]);
                                    const float a = __uint_as_float(r[8 * q + 2 * h + e]);
                                    const float sg = __fdividef(1.f, 1.f + __expf(-x));
                                    const float xs = x * sg;  // silu(g)
                                    wdot = __fmaf_rn(a, xs * uu, wdot);
                                    const float d = a * wrow;
                                    du2[e] = xs * d;
                                    dg2[e] = uu * d * (sg * (1.f + x * (1.f - sg)));
                                }
                                dgp[4 * q + h] = pack_bf16(dg2[0], dg2[1]);
                                dup[4 * q + h] = pack_bf16(du2[0], du2[1]);
                            }
                        }
                        // (measured: TMA-staged stores beat direct register->global stores here,
                        // 0.57 vs 0.61 ms per dgrad at config B)
                        stg.put2d_packed(&p.mapO0, lane, dgp, col, ti.m0 + row0);
                        stg.put2d_packed(&p.mapO0, lane, dup, p.I + col, ti.m0 + row0);
                        if (wscheme && (col & 63) == 32) {  // end of a 64-column weight-gradient slot
                            p.wpart[(int64_t)(ti.m0 + row0 + lane) * (p.I / 64) + col / 64] = wdot;
                            wdot = 0.f;
                        }
                    }
                } else if constexpr (KIND == GemmKind::FwdGateUp) {
                    const int nbase = ti.n0 / 2;  // 128 gate + 128 up columns per tile
                    uint32_t r[32], r2[32];
    #pragma unroll 1
                    for (int c = half * (BN / 4); c < (half + 1) * (BN / 4); c += 32) {
                        tmem_ld32(tacc + c, r);
                        tmem_ld32(tacc + BN / 2 + c, r2);
                        tmem_wait_ld();
                        const int col = nbase + c;
                        if (col >= p.I) continue;  // I % 64 == 0: all in or all out
                        float gv[32], uv[32], hv[32];
                        // G and U are stored rounded to bf16; H is computed from the rounded values
    #pragma unroll
                        for (int j = 0; j < 32; j += 2) {
                            const uint32_t gp = pack_bf16(__uint_as_float(r[j]), __uint_as_float(r[j + 1]));
                            const uint32_t up = pack_bf16(__uint_as_float(r2[j]), __uint_as_float(r2[j + 1]));
                            gv[j] = bf16_lo(gp);
                            gv[j + 1] = bf16_hi(gp);
                            uv[j] = bf16_lo(up);
                            uv[j + 1] = bf16_hi(up);
                        }
    #pragma unroll
                        for (int j = 0; j < 32; ++j) hv[j] = silu_f(gv[j]) * uv[j] * wrow;
                        stg.put2d(&p.mapO0, lane, gv, col, ti.m0 + row0);
                        stg.put2d(&p.mapO1, lane, uv, col, ti.m0 + row0);
                        stg.put2d(&p.mapO2, lane, hv, col, ti.m0 + row0);
                    }
                } else if constexpr (KIND == GemmKind::FwdDown || KIND == GemmKind::BwdDx) {
                    uint32_t r[32];
                    float v[32];
    #pragma unroll 1
                    for (int c = half * (BN / 2); c < (half + 1) * (BN / 2); c += 32) {
                        tmem_ld32(tacc + c, r);
                        tmem_wait_ld();
                        const int col = ti.n0 + c;
                        if (col >= p.H) continue;
    #pragma unroll
                        for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
                        stg.put2d(&p.mapO0, lane, v, col, ti.m0 + row0);
                    }
                } else if constexpr (KIND == GemmKind::WgradDown || KIND == GemmKind::WgradGateUp) {
                    // out[e][m][n] * scale through 3-D maps: rows past the expert's M are clipped
                    uint32_t r[32];
                    float v[32];
                    const bool zero = ti.kb == 0;
    #pragma unroll 1
                    for (int c = half * (BN / 2); c < (half + 1) * (BN / 2); c += 32) {
                        if (!zero) {
                            tmem_ld32(tacc + c, r);
                            tmem_wait_ld();
                        }
    #pragma unroll
                        for (int j = 0; j < 32; ++j) v[j] = zero ? 0.f : __uint_as_float(r[j]) * p.scale;
                        const int col = ti.n0 + c;
                        if constexpr (KIND == GemmKind::WgradDown) {
                            if (col < p.H) stg.put3d(&p.mapO0, lane, v, col, ti.m0 + row0, ti.e);
                        } else {
                            if (col < p.I) stg.put3d(&p.mapO0, lane, v, col, ti.m0 + row0, ti.e);
                            else if (col < 2 * p.I) stg.put3d(&p.mapO1, lane, v, col - p.I, ti.m0 + row0, ti.e);
                        }
                    }
                } else {
                    epilogue_tile<KIND>(p, ti, tacc, 32 * quad + lane, ti.kb == 0, half);
                }
            };
            auto release = [&](int a) {  // this warp is done reading accumulator (half) a
                tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    if constexpr (CG == 1) mbar_arrive(tempty_bar(a));
                    else mbar_arrive_cluster(tempty0 + 8u * a);
                }
            };
            if constexpr (KC::WIDE && (KIND == GemmKind::FwdDown || KIND == GemmKind::BwdDx ||
                                       KIND == GemmKind::WgradDown || KIND == GemmKind::WgradGateUp)) {
                // a half leaves TMEM first (this warp's 32 rows x 128 columns, packed to bf16 in
                // registers), is released to the next tile's MMAs, and only then goes out through the
                // staging slots — the stores no longer hold the accumulator
                constexpr bool kWgrad = KIND == GemmKind::WgradDown || KIND == GemmKind::WgradGateUp;
                const bool zero = kWgrad && ti.kb == 0;  // empty expert: zero weight gradient
                const float sc = kWgrad ? p.scale : 1.f;
#pragma unroll 1
                for (int hh = 0; hh < KC::REGIONS; ++hh) {
                    uint32_t pk[4][16];
#pragma unroll
                    for (int ch = 0; ch < 4; ch += 2) {
                        uint32_t r0[32], r1[32];
                        if (!zero) {
                            tmem_ld32(tacc0 + BN * hh + half * (BN / 2) + 32 * ch, r0);
                            tmem_ld32(tacc0 + BN * hh + half * (BN / 2) + 32 * (ch + 1), r1);
                            tmem_wait_ld();
                        }
#pragma unroll
                        for (int j = 0; j < 16; ++j) {
                            pk[ch][j] = zero ? 0u : pack_bf16(__uint_as_float(r0[2 * j]) * sc, __uint_as_float(r0[2 * j + 1]) * sc);
                            pk[ch + 1][j] =
                                zero ? 0u : pack_bf16(__uint_as_float(r1[2 * j]) * sc, __uint_as_float(r1[2 * j + 1]) * sc);
                        }
                    }
                    release(hh);
#pragma unroll
                    for (int ch = 0; ch < 4; ++ch) {
                        const int col = ti.n0 + BN * hh + half * (BN / 2) + 32 * ch;
                        if constexpr (KIND == GemmKind::FwdDown || KIND == GemmKind::BwdDx) {
                            if (col < p.H) stg.put2d_packed(&p.mapO0, lane, pk[ch], col, ti.m0 + row0);
                        } else if constexpr (KIND == GemmKind::WgradDown) {
                            if (col < p.H) stg.put3d_packed(&p.mapO0, lane, pk[ch], col, ti.m0 + row0, ti.e);
                        } else {
                            if (col < p.I) stg.put3d_packed(&p.mapO0, lane, pk[ch], col, ti.m0 + row0, ti.e);
                            else if (col < 2 * p.I)
                                stg.put3d_packed(&p.mapO1, lane, pk[ch], col - p.I, ti.m0 + row0, ti.e);
                        }
                    }
                }
            } else if constexpr (KC::WIDE && KIND == GemmKind::FwdGateUp) {
                // per region: this warp's two gate chunks and their up chunks leave TMEM rounded to
                // bf16 (what is stored; H is computed from the rounded values), the region is released,
                // then G, U and H' = w * silu(G) * U go out through the staging slots
#pragma unroll 1
                for (int hh = 0; hh < KC::REGIONS; ++hh) {
                    uint32_t gp[2][16], up[2][16];
#pragma unroll
                    for (int ch = 0; ch < 2; ++ch) {
                        uint32_t r[32], r2[32];
                        const int c = half * (BN / 4) + 32 * ch;
                        tmem_ld32(tacc0 + BN * hh + c, r);
                        tmem_ld32(tacc0 + BN * hh + BN / 2 + c, r2);
                        tmem_wait_ld();
#pragma unroll
                        for (int j = 0; j < 16; ++j) {
                            gp[ch][j] = pack_bf16(__uint_as_float(r[2 * j]), __uint_as_float(r[2 * j + 1]));
                            up[ch][j] = pack_bf16(__uint_as_float(r2[2 * j]), __uint_as_float(r2[2 * j + 1]));
                        }
                    }
                    release(hh);
#pragma unroll
                    for (int ch = 0; ch < 2; ++ch) {
                        const int col = (ti.n0 + BN * hh) / 2 + half * (BN / 4) + 32 * ch;
                        if (col >= p.I) continue;  // I % 64 == 0: all in or all out
                        uint32_t hp[16];
#pragma unroll
                        for (int j = 0; j < 16; ++j) {
                            const float g0 = bf16_lo(gp[ch][j]), g1 = bf16_hi(gp[ch][j]);
                            const float u0 = bf16_lo(up[ch][j]), u1 = bf16_hi(up[ch][j]);
                            hp[j] = pack_bf16(silu_f(g0) * u0 * wrow, silu_f(g1) * u1 * wrow);
                        }
                        stg.put2d_packed(&p.mapO0, lane, gp[ch], col, ti.m0 + row0);
                        stg.put2d_packed(&p.mapO1, lane, up[ch], col, ti.m0 + row0);
                        stg.put2d_packed(&p.mapO2, lane, hp, col, ti.m0 + row0);
                    }
                }
            } else if constexpr (KC::WIDE) {
#pragma unroll 1
                for (int hh = 0; hh < KC::REGIONS; ++hh) {
                    TileInfo th = ti;
                    th.n0 += BN * hh;
                    drain(tacc0 + BN * hh, th);
                    release(hh);
                }
            } else {
                drain(tacc0, ti);
                release(acc);
            }

        }
        if constexpr (KC::TMA_EPI) stg.drain(lane);  // the bulk stores have left shared memory
    }
    tc_fence_before();
    if constexpr (CG == 2) cluster_sync_all();
    else __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        if constexpr (CG == 1)
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS)
                         : "memory");
        else
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS)
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
static CUtensorMap make_map(const void* ptr, int64_t cols, int64_t rows, int bc, int br,
                            CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
    CUtensorMap m;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)std::max<int64_t>(rows, 1)};
    cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
    cuuint32_t box[2] = {(cuuint32_t)bc, (cuuint32_t)br};
    cuuint32_t es[2] = {1, 1};
    CUresult r = get_encode()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, es,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
    return m;
}

// 3-D bf16 tensor [d2][d1][d0] (d0 contiguous), box {32, 32, 1}, 64B swizzle: the TMA-store
// view of a weight gradient, whose rows past d1 (a partial M tile) are clipped by the engine
static CUtensorMap make_map3(const void* ptr, int64_t d0, int64_t d1, int64_t d2) {
    CUtensorMap m;
    cuuint64_t dims[3] = {(cuuint64_t)d0, (cuuint64_t)d1, (cuuint64_t)std::max<int64_t>(d2, 1)};
    cuuint64_t strides[2] = {(cuuint64_t)d0 * 2, (cuuint64_t)(d0 * d1) * 2};
    cuuint32_t box[3] = {32, 32, 1};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = get_encode()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), dims, strides, box, es,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                              CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled (3d) failed: " + std::to_string((int)r));
    return m;
}
static CUtensorMap make_store_map(const void* ptr, int64_t cols, int64_t rows) {
    return make_map(ptr, cols, rows, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B);
}

template <GemmKind KIND, int CG>
static void launch_kind(const Params& p, int grid, cudaStream_t st) {
    static std::once_flag once;
    static int max_clusters = 0;  // co-resident clusters of CG CTAs (GPC packing)
    constexpr int smem = KCfg<KIND, CG>::SMEM;
    std::call_once(once, [] {
        B2_CUDA(cudaFuncSetAttribute(grouped_gemm_kernel<KIND, CG>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        cudaLaunchConfig_t q{};
        q.gridDim = dim3(148);
        q.blockDim = dim3(NUM_THREADS);
        q.dynamicSmemBytes = smem;
        cudaLaunchAttribute ca[1];
        ca[0].id = cudaLaunchAttributeClusterDimension;
        ca[0].val.clusterDim.x = CG;
        ca[0].val.clusterDim.y = 1;
        ca[0].val.clusterDim.z = 1;
        q.attrs = ca;
        q.numAttrs = 1;
        if (cudaOccupancyMaxActiveClusters(&max_clusters, grouped_gemm_kernel<KIND, CG>, &q) != cudaSuccess) {
            cudaGetLastError();
            max_clusters = 0;
        }
    });
    if (max_clusters > 0) grid = std::min(grid, max_clusters * CG);
    grid = std::max(CG, grid / CG * CG);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(NUM_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CG;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    B2_CUDA(cudaLaunchKernelEx(&cfg, grouped_gemm_kernel<KIND, CG>, p));
}

}  // namespace sm100

int router_dw_splits(int64_t S, int64_t H, int num_sms) {
    const int64_t mt = ceil_div(H, sm100::BM);
    const int64_t want = std::max<int64_t>(1, (num_sms > 0 ? num_sms : 148) / mt);
    const int64_t max_by_rows = std::max<int64_t>(1, ceil_div(std::max<int64_t>(S, 1), 256));
    return (int)std::min<int64_t>(std::min<int64_t>(want, max_by_rows), kRouterDwMaxSplits);
}

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
    p.row_w = a.row_w;
    p.wpart = a.wpart;
    p.eorder = a.expert_order;
    if (a.kind == GemmKind::BwdDownDgrad && a.row_w) check(a.wpart != nullptr, "dgrad: row weights need wpart");
    const int64_t P = a.pmax, H = a.H, I = a.I, nr = a.nr;
    int grid = a.num_sms > 0 ? a.num_sms : 148;
    if (a.max_ctas > 0) grid = std::min(grid, std::max(2, a.max_ctas));
    p.umma_n = BN;
    p.b_chunks = 4;
    p.S = a.S;
    p.N = a.N;
    p.counts = a.counts;
    // the six expert GEMMs run as 256 x 256 tiles on CTA pairs (cta_group::2)
    constexpr int G = 2;
    using C2 = Cfg<G>;
    p.stage_tx = G * C2::STAGE_BYTES;
    switch (a.kind) {
        case GemmKind::FwdGateUp:
        case GemmKind::FwdDown:
            p.idesc = umma_idesc(false, true, BN, BM * G);
            break;
        case GemmKind::BwdDownDgrad:
        case GemmKind::BwdDx:
            p.idesc = umma_idesc(false, false, BN, BM * G);
            break;
        case GemmKind::RouterDx:
            p.idesc = umma_idesc(false, false);
            p.stage_tx = Cfg<1>::STAGE_BYTES;
            break;
        default:
            p.idesc = umma_idesc(true, true, BN, BM * G);
            break;
    }
    switch (a.kind) {
        case GemmKind::FwdGateUp: {
            using K0 = KCfg<GemmKind::FwdGateUp, G>;
            p.n_tiles = (int)ceil_div(I, K0::TN / 2);
            p.stage_tx = G * K0::STAGE_BYTES;
            p.mapA = make_map(a.x, H, P, 64, BM);
            p.mapB0 = make_map(a.wg, I, nr * H, 64, 64);
            p.mapB1 = make_map(a.wu, I, nr * H, 64, 64);
            p.mapO0 = make_store_map(a.out0, I, P);
            p.mapO1 = make_store_map(a.out1, I, P);
            p.mapO2 = make_store_map(a.out2, I, P);
            p.num_kb_fixed = (int)ceil_div(H, BK);
            launch_kind<GemmKind::FwdGateUp, G>(p, grid, st);
            break;
        }
        case GemmKind::FwdDown: {
            using K1 = KCfg<GemmKind::FwdDown, G>;
            p.n_tiles = (int)ceil_div(H, K1::TN);
            p.stage_tx = G * K1::STAGE_BYTES;
            p.mapA = make_map(a.h, I, P, 64, BM);
            p.mapB0 = make_map(a.wd, H, nr * I, 64, 64);
            p.mapB1 = p.mapB0;
            p.mapO0 = make_store_map(a.out0, H, P);
            p.num_kb_fixed = (int)ceil_div(I, BK);
            launch_kind<GemmKind::FwdDown, G>(p, grid, st);
            break;
        }
        case GemmKind::BwdDownDgrad: {
            using K2 = KCfg<GemmKind::BwdDownDgrad, G>;
            p.n_tiles = (int)ceil_div(I, K2::TN);
            p.stage_tx = G * K2::STAGE_BYTES;
            p.mapA = make_map(a.dy, H, P, 64, BM);
            p.mapB0 = make_map(a.wd, H, nr * I, 64, C2::B_COLS);
            p.mapB1 = p.mapB0;
            p.mapO0 = make_store_map(a.out0, 2 * I, P);
            p.num_kb_fixed = (int)ceil_div(H, BK);
            launch_kind<GemmKind::BwdDownDgrad, G>(p, grid, st);
            break;
        }
        case GemmKind::BwdDx: {
            using K3 = KCfg<GemmKind::BwdDx, G>;
            p.n_tiles = (int)ceil_div(H, K3::TN);
            p.stage_tx = G * K3::STAGE_BYTES;
            p.mapA = make_map(a.dgu, 2 * I, P, 64, BM);
            p.mapB0 = make_map(a.wg, I, nr * H, 64, C2::B_COLS);
            p.mapB1 = make_map(a.wu, I, nr * H, 64, C2::B_COLS);
            p.mapO0 = make_store_map(a.out0, H, P);
            p.num_kb_fixed = (int)ceil_div(2 * I, BK);
            launch_kind<GemmKind::BwdDx, G>(p, grid, st);
            break;
        }
        case GemmKind::WgradDown: {
            check(a.counts != nullptr, "wgrad: expert row counts required");
            p.mapA = make_map(a.h, I, P, 64, 64);
            p.mapB0 = make_map(a.dy, H, P, 64, 64);
            p.mapB1 = p.mapB0;
            p.mapO0 = make_map3(a.out0, H, I, nr);
            p.m_tiles_fixed = (int)ceil_div(I, BM * G);
            p.n_tiles = (int)ceil_div(H, KCfg<GemmKind::WgradDown, G>::TN);
            p.stage_tx = G * KCfg<GemmKind::WgradDown, G>::STAGE_BYTES;
            grid = (int)std::min<int64_t>(grid, G * nr * p.m_tiles_fixed * p.n_tiles);
            launch_kind<GemmKind::WgradDown, G>(p, grid, st);
            break;
        }
        case GemmKind::WgradGateUp: {
            check(a.counts != nullptr, "wgrad: expert row counts required");
            p.mapA = make_map(a.x, H, P, 64, 64);
            p.mapB0 = make_map(a.dgu, 2 * I, P, 64, 64);
            p.mapB1 = p.mapB0;
            p.mapO0 = make_map3(a.out0, I, H, nr);
            p.mapO1 = make_map3(a.out1, I, H, nr);
            p.m_tiles_fixed = (int)ceil_div(H, BM * G);
            p.n_tiles = (int)ceil_div(2 * I, KCfg<GemmKind::WgradGateUp, G>::TN);
            p.stage_tx = G * KCfg<GemmKind::WgradGateUp, G>::STAGE_BYTES;
            grid = (int)std::min<int64_t>(grid, G * nr * p.m_tiles_fixed * p.n_tiles);
            launch_kind<GemmKind::WgradGateUp, G>(p, grid, st);
            break;
        }
        case GemmKind::RouterDx: {
            check(a.N % 8 == 0 && a.N <= 256, "router dx GEMM: n_experts must be a multiple of 8, <= 256");
            const int64_t S = a.S;
            if (S <= 0) return;
            check(a.dl_lo != nullptr, "router dx GEMM: needs the low half of the dlogits split");
            p.mapA = make_map(a.dl, a.N, S, 64, BM);
            p.mapA1 = make_map(a.dl_lo, a.N, S, 64, BM);
            p.mapB0 = make_map(a.wr, a.N, H, 64, BN);
            p.mapB1 = p.mapB0;
            p.n_tiles = (int)ceil_div(H, BN);
            p.num_kb_fixed = 2 * (int)ceil_div(a.N, BK);  // hi then lo
            p.src = (const __nv_bfloat16*)a.src;
            grid = (int)std::min<int64_t>(grid, ceil_div(S, BM) * p.n_tiles);
            launch_kind<GemmKind::RouterDx, 1>(p, grid, st);
            break;
        }
        case GemmKind::RouterDw: {
            check(a.N % 8 == 0 && a.N <= 256, "router dW GEMM: n_experts must be a multiple of 8, <= 256");
            const int64_t S = a.S;
            p.umma_n = (int)round_up(a.N, 16);
            p.idesc = umma_idesc(true, true, p.umma_n);
            p.b_chunks = (int)ceil_div(a.N, 64);
            p.stage_tx = A_BYTES + 8192u * p.b_chunks;
            p.mapA = make_map(a.x, H, std::max<int64_t>(S, 1), 64, 64);
            p.mapB0 = make_map(a.dl, a.N, std::max<int64_t>(S, 1), 64, 64);
            p.mapB1 = p.mapB0;
            p.m_tiles_fixed = (int)ceil_div(H, BM);
            p.n_tiles = 1;
            const int nsplit = router_dw_splits(S, H, a.num_sms);
            p.rows_per_split = (int)round_up(ceil_div(std::max<int64_t>(S, 1), nsplit), BK);
            p.nr = nsplit;  // tiles = nsplit * m_tiles
            p.part = a.part;
            grid = (int)std::min<int64_t>(grid, (int64_t)nsplit * p.m_tiles_fixed);
            launch_kind<GemmKind::RouterDw, 1>(p, grid, st);
            break;
        }
    }
}

}  // namespace b2
