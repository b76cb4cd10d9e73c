"""Real-run kernel timeline of the bench step (CUPTI via torch.profiler, no ncu
serialisation): per-kernel average duration, share of the step, and idle gaps.
Usage: python tools/timeline.py [--steps 3] [--graph]"""
import argparse
import collections
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--graph", action="store_true")
    ap.add_argument("--tokens", type=int, default=16384)
    ap.add_argument("--no-overlap", action="store_true", help="EP: dX return after the wgrad GEMMs")
    args = ap.parse_args()
    import torch
    from torch.profiler import ProfilerActivity, profile

    import paper_2604_00785_b200 as b2
    H, N, K, I, S = 2048, 64, 8, 1024, args.tokens
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    dev = torch.device("cuda", rank)
    torch.cuda.set_device(dev)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    nccl_id = None
    if world > 1:  # EP = world over NVLink peer memory (launch with torchrun)
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
        ids = [b2.Context.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(ids, src=0)
        nccl_id = ids[0]
    ctx = b2.Context(rank, rank=rank, ep=world, nccl_id=nccl_id, stream=stream)
    cfg = b2.MoeConfig(n_experts=N, top_k=K, hidden=H, intermediate=I, ep=world)
    gen = torch.Generator(device=dev).manual_seed(1234 + rank)
    mk = lambda shape, std: (torch.randn(shape, device=dev, generator=gen) * std).bfloat16()
    NR = N // world
    router = (torch.randn((H, N), device=dev, generator=torch.Generator(device=dev).manual_seed(7)) * 0.02).bfloat16()
    gate, up, down = mk((NR, H, I), 0.02), mk((NR, H, I), 0.02), mk((NR, I, H), 0.02)
    x, dout = mk((S, H), 1.0), mk((S, H), 1.0)
    layer = b2.MoeLayer(ctx, cfg, torch.bfloat16, S)
    if args.graph:
        layer.set_graph(True)
    if args.no_overlap:
        import ctypes
        b2.lib().b2x_moe_set_overlap_return.argtypes = [ctypes.c_void_p, ctypes.c_int]
        b2.lib().b2x_moe_set_overlap_return(layer.h, 0)
    out = torch.empty_like(x)
    grads = dict(input=torch.empty_like(x), router=torch.empty_like(router), gate=torch.empty_like(gate),
                 up=torch.empty_like(up), down=torch.empty_like(down))
    apg = torch.empty((S, N), dtype=torch.float32, device=dev)

    def step():
        layer.forward(x, router, gate, up, down, out=out)
        layer.aux_probs_grad(0.01, out=apg)
        layer.backward(router, gate, up, down, dout, apg, grads=grads)

    for _ in range(5):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(10):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    if rank == 0:
        print(f"event-timed step: {e0.elapsed_time(e1) / 10:.3f} ms (EP={world})")
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(args.steps):
            step()
        torch.cuda.synchronize()
    ev = [e for e in prof.events() if e.device_type.name == "CUDA" and e.time_range.elapsed_us() > 0]
    ev.sort(key=lambda e: e.time_range.start)
    if world > 1:  # per-rank view of the EP barriers (time spent waiting = skew between ranks)
        bars = [e.time_range.elapsed_us() for e in ev if "flag_barrier" in e.name]
        gemm = sum(e.time_range.elapsed_us() for e in ev if "grouped_gemm" in e.name) / args.steps
        nb = max(1, len(bars) // args.steps)
        per = [sum(bars[i::nb]) / args.steps for i in range(nb)]
        print(f"rank {rank}: barrier waits per step (in order) {' '.join(f'{b:7.1f}' for b in per)} us; "
              f"GEMMs {gemm / 1e3:.3f} ms/step", flush=True)
    if rank != 0:
        return
    agg = collections.defaultdict(list)
    for e in ev:
        agg[e.name.split("(")[0][:70]].append(e.time_range.elapsed_us())
    span = ev[-1].time_range.end - ev[0].time_range.start
    busy = sum(e.time_range.elapsed_us() for e in ev)
    gaps = []
    for a, b in zip(ev, ev[1:]):
        g = b.time_range.start - a.time_range.end
        if g > 0:
            gaps.append((g, a.name.split("(")[0][:40], b.name.split("(")[0][:40]))
    print(f"span {span / args.steps / 1e3:.3f} ms/step, kernel busy {busy / args.steps / 1e3:.3f} ms/step")
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        print(f"{sum(v) / busy * 100:5.1f}% {len(v) // args.steps:3d}/step {sum(v) / len(v):9.1f} us  {k}")
    gaps.sort(reverse=True)
    print("largest gaps (us):")
    for g in gaps[:12]:
        print(f"  {g[0]:8.1f}  {g[1]} -> {g[2]}")
    print(f"total gap {sum(g[0] for g in gaps) / args.steps:.1f} us/step over {len(gaps)} gaps")


if __name__ == "__main__":
    main()
