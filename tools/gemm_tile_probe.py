#!/usr/bin/env python
"""Times one grouped-GEMM kind (b2x_grouped_gemm) on synthetic expert groups of given row counts,
to see what a 256-row tile and a 128-row half tile cost (config B dims: H 2048, I 1024).

  python tools/gemm_tile_probe.py --kind 1 --rows 256 384 128
"""
import argparse
import ctypes as C
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2604_00785_b200 as b2  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kind", type=int, default=1)
    ap.add_argument("--rows", type=int, nargs="+", default=[256, 384, 128])
    ap.add_argument("--experts", type=int, default=64)
    ap.add_argument("--H", type=int, default=2048)
    ap.add_argument("--I", type=int, default=1024)
    ap.add_argument("--iters", type=int, default=20)
    a = ap.parse_args()
    lib = b2.lib()
    fn = lib.b2x_grouped_gemm
    fn.restype = C.c_int
    fn.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_int64] + \
        [C.c_void_p] * 12 + [C.c_float]
    ctx = b2.Context(0)
    H, I, nr = a.H, a.I, a.experts
    p = lambda t: C.c_void_p(t.data_ptr())
    for rows in a.rows:
        starts = [e * ((rows + 127) // 128 * 128) for e in range(nr + 1)]
        P = starts[-1] + 256
        ps = torch.tensor(starts, dtype=torch.int32, device="cuda")
        cnt = torch.full((nr,), rows, dtype=torch.int32, device="cuda")
        mk = lambda *s: (torch.randn(*s, device="cuda") * 0.05).bfloat16()
        x, g, u, h, dy, dgu = mk(P, H), mk(P, I), mk(P, I), mk(P, I), mk(P, H), mk(P, 2 * I)
        wg, wu, wd = mk(nr, H, I), mk(nr, H, I), mk(nr, I, H)
        o0 = torch.empty(P, 2 * max(H, I), dtype=torch.bfloat16, device="cuda")
        o1, o2 = torch.empty_like(o0), torch.empty_like(o0)
        if a.kind in (4, 5):
            o0 = torch.empty(nr, max(H, I), max(H, I), dtype=torch.bfloat16, device="cuda")
            o1 = torch.empty_like(o0)

        def run():
            rc = fn(ctx.h, a.kind, H, I, nr, p(ps), p(cnt), P, p(x), p(wg), p(wu), p(wd), p(g), p(u), p(h), p(dy),
                    p(dgu), p(o0), p(o1), p(o2), 1.0)
            assert rc == 0, lib.b2_last_error()

        for _ in range(3):
            run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.iters):
            run()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.iters
        flop = {0: 4, 1: 2, 2: 2, 3: 4, 4: 2, 5: 4}[a.kind] * nr * rows * H * I
        print(f"kind {a.kind} rows/expert {rows:5d}: {ms * 1e3:8.1f} us  {flop / ms / 1e9:7.1f} TFLOP/s (useful rows)")


if __name__ == "__main__":
    main()
