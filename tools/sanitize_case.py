#!/usr/bin/env python
"""A small workload for compute-sanitizer (memcheck / racecheck / synccheck / initcheck): one
bf16 (tcgen05) and one fp32 MoE layer forward + backward, the routing-artifact export and a
sharded AdamW step, all eager on cuda:0 — every hot-path kernel launches at least once.
With torchrun (WORLD_SIZE = 2) it runs the EP = 2 layer instead (NVLink peer memory, flag
barriers). tools/sanitize.sh drives it."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2604_00785_b200 as b2  # noqa: E402


def layer_step(ctx, dt, ep=1, rank=0, S=256, H=256, I=128, N=16, K=4):
    cfg = b2.MoeConfig(n_experts=N, top_k=K, hidden=H, intermediate=I, ep=ep)
    g = torch.Generator(device="cuda").manual_seed(5 + rank)
    mk = lambda *s: (torch.randn(*s, device="cuda", generator=g) * 0.05).to(dt)
    nr = N // ep
    x, dout = mk(S, H) * 20, mk(S, H) * 20
    router = (torch.randn(H, N, device="cuda", generator=torch.Generator(device="cuda").manual_seed(1)) * 0.05).to(dt)
    gate, up, down = mk(nr, H, I), mk(nr, H, I), mk(nr, I, H)
    layer = b2.MoeLayer(ctx, cfg, dt, S)
    out = layer.forward(x, router, gate, up, down)
    grads = layer.backward(router, gate, up, down, dout, layer.aux_probs_grad(0.01))
    torch.cuda.synchronize()
    layer.artifacts()
    assert torch.isfinite(out.float()).all() and torch.isfinite(grads["input"].float()).all()
    layer.close()


def main():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    torch.cuda.set_device(rank)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")
        ids = [b2.Context.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(ids, src=0)
        ctx = b2.Context(rank, rank=rank, ep=world, nccl_id=ids[0])
        layer_step(ctx, torch.bfloat16, ep=world, rank=rank)
        dist.barrier()
        ctx.close()
        print(f"rank {rank}: EP={world} layer ok")
        return
    ctx = b2.Context(0)
    layer_step(ctx, torch.bfloat16)
    layer_step(ctx, torch.float32, S=96, H=64, I=48, N=8, K=2)
    n = 70_000
    W = (torch.randn(n, device="cuda") * 0.02).bfloat16()
    G = (torch.randn(n, device="cuda") * 1e-3).bfloat16()
    opt = b2.ShardedOptimizer(ctx, b2.AdamWConfig(warmup_steps=0), [(W[:50_000], G[:50_000], 1, 0),
                                                                     (W[50_000:], G[50_000:], 0, 0)], b2.EPSO)
    opt.step()
    torch.cuda.synchronize()
    print("sanitize case ok")


if __name__ == "__main__":
    main()
