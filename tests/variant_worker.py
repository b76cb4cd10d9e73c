"""One process of the kernel-variant equivalence test (tests/test_gpu_variants.py).

The opt-in A/B hooks (B2_GEMM_MC, B2_LOGITS_IMPL, B2_ADAMW_IMPL) are read once per process, so
each variant runs here in its own process: a bf16 MoE layer forward + backward and two sharded
AdamW steps on fixed seeded inputs, every output saved to an .npz for a bitwise comparison.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main(out_path):
    import torch

    import paper_2604_00785_b200 as b2
    torch.manual_seed(0)
    ctx = b2.Context(0)
    # H = 512, I = 256: every expert GEMM kind except the dgrad has an even number of N tiles, so
    # the two-pair multicast clusters are exercised; S not a multiple of the 32-token logits tile
    kw = dict(n_experts=16, top_k=4, hidden=512, intermediate=256)
    cfg = b2.MoeConfig(**kw)
    S, H, I, N = 1000, 512, 256, 16
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(1)
    mk = lambda shape, std: (torch.randn(shape, device=dev, generator=g) * std).bfloat16()
    router, gate, up, down = mk((H, N), 0.05), mk((N, H, I), 0.02), mk((N, H, I), 0.02), mk((N, I, H), 0.02)
    x, dout = mk((S, H), 1.0), mk((S, H), 1.0)
    layer = b2.MoeLayer(ctx, cfg, torch.bfloat16, S)
    out = layer.forward(x, router, gate, up, down)
    grads = layer.backward(router, gate, up, down, dout)
    torch.cuda.synchronize()
    res = {"out": out, **{f"d_{k}": v for k, v in grads.items()}}
    # sharded AdamW (bf16 grads and weights, the vectorised path), two steps
    n = 3 * 4096 + 8
    w = (torch.randn(n, device=dev, generator=g) * 0.05).bfloat16()
    gr = (torch.randn(n, device=dev, generator=g) * 1e-3).bfloat16()
    opt = b2.ShardedOptimizer(ctx, b2.AdamWConfig(warmup_steps=0), [(w, gr, 0, 0)], b2.EPSO)
    opt.step()
    opt.step()
    torch.cuda.synchronize()
    res["adamw_w"] = w
    master, m, v = opt.state(0)
    np.savez(out_path, **{k: (t.float().cpu().numpy() if hasattr(t, "cpu") else t) for k, t in res.items()},
             master=master, m=m, v=v)


if __name__ == "__main__":
    main(sys.argv[1])
