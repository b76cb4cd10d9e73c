"""Profiling probe: the fused AdamW shard kernel on a 1 Gi-element bf16 slot (one GPU)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2604_00785_b200 as b2

n = int(sys.argv[1]) if len(sys.argv) > 1 else (1 << 30)
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
ctx = b2.Context(0)
w = (torch.randn(n, device="cuda") * 0.02).bfloat16()
g = (torch.randn(n, device="cuda") * 1e-3).bfloat16()
opt = b2.ShardedOptimizer(ctx, b2.AdamWConfig(warmup_steps=0), [(w, g, 1, 0)], b2.EPSO)
for _ in range(2):
    opt.step(stats=False)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(steps):
    opt.step(stats=False)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / steps
print(f"adamw n={n} {ms:.3f} ms/step  {n * 30 / ms / 1e6:.1f} GB/s (30 B/elem incl. norm pass)")
