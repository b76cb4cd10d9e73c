#!/usr/bin/env python
"""Times the router (logits + softmax/top-k, b2_route) at config B: python tools/logits_probe.py"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2604_00785_b200 as b2  # noqa: E402


def main(S=16384, H=2048, N=64, K=8, iters=50):
    ctx = b2.Context(0)
    cfg = b2.MoeConfig(n_experts=N, top_k=K, hidden=H, intermediate=1024)
    x = torch.randn(S, H, device="cuda").bfloat16()
    w = (torch.randn(H, N, device="cuda") * 0.02).bfloat16()
    for _ in range(3):
        b2.route(ctx, cfg, x, w)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        out = b2.route(ctx, cfg, x, w)
    e1.record()
    torch.cuda.synchronize()
    print(f"route (logits + softmax/top-k) S={S} H={H} N={N}: {e0.elapsed_time(e1) / iters * 1e3:.1f} us "
          f"(incl. output allocation); logits checksum {out[0].double().sum().item():.6e}")


if __name__ == "__main__":
    main()
