"""EPSO step on a synthetic parameter set (one process, one GPU) for ncu captures and
quick timing: python tools/adamw_probe.py [--gelems 1.0] [--steps 5]"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gelems", type=float, default=1.0)
    ap.add_argument("--steps", type=int, default=5)
    args = ap.parse_args()
    import torch

    import paper_2604_00785_b200 as b2
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = b2.Context(0, stream=stream)
    n = int(args.gelems * 1e9)
    third = (n // 3) // 64 * 64  # multiples of 64: every slot takes the vectorised path, as the Mula set does
    sizes = [third, third, n - 2 * third]
    ws = [(torch.randn(k, device="cuda") * 0.02).bfloat16() for k in sizes]
    gs = [(torch.randn(k, device="cuda") * 1e-3).bfloat16() for k in sizes]
    opt = b2.ShardedOptimizer(ctx, b2.AdamWConfig(warmup_steps=0), [(w, g, 1, 0) for w, g in zip(ws, gs)], b2.EPSO)
    for _ in range(2):
        opt.step(stats=False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        opt.step(stats=False)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    print(f"{n / 1e9:.2f} G elements: {ms:.3f} ms/step, {30 * n / ms / 1e6:.0f} GB/s algorithmic (30 B/elem)")


if __name__ == "__main__":
    main()
