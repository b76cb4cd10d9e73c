/*
 * b2moe_testing.h — unit-test hooks of libb2moe.so (not part of the drop-in
 * boundary). They run one stage of the hot path in isolation so the tests can
 * check each kernel against a reference of the same op.
 */
#ifndef B2MOE_TESTING_H
#define B2MOE_TESTING_H
#include "b2moe.h"
#ifdef __cplusplus
extern "C" {
#endif
/* One tcgen05 grouped GEMM of the expert MLP (kind: 0 FwdGateUp, 1 FwdDown,
 * 2 BwdDownDgrad, 3 BwdDx, 4 WgradDown, 5 WgradGateUp), bf16 operands in the
 * padded expert-row layout; pad_start [nr+1] int32 device (multiples of 256),
 * counts [nr] int32 device rows per expert. */
int b2x_grouped_gemm(b2_ctx* ctx, int kind, int hidden, int intermediate, int nr, const int32_t* pad_start,
                     const int32_t* counts, int64_t pmax, const void* x, const void* wg, const void* wu, const void* wd, const void* g,
                     const void* u, const void* h, const void* dy, const void* dgu, void* out0, void* out1,
                     void* out2, float scale);
/* EP >= 4, bf16: overlap (1, default) the backward's dX return with the weight-gradient
 * GEMMs (side stream, GEMM grid reduced by 32 SMs) or run it after them (0); at EP 2 the
 * return always runs after them (measured faster). */
int b2x_moe_set_overlap_return(b2_moe* m, int on);
#ifdef __cplusplus
}
#endif
#endif
