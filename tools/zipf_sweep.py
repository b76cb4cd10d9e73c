"""Config E sweep (BASELINE.md load-imbalance line): the Mula-20B-A2B-shaped layer
(H 2048, 96 experts top-8, ffn 1024, 16,384 tokens per GPU) under Zipf routing s ∈ {0, 1.0, 1.2},
identity and seeded-random expert permutation, EP = world. One JSON line per case (rank 0):
tokens/s and the max/mean rows per rank.
    torchrun --nproc-per-node 4 --master-addr 127.0.0.1 tools/zipf_sweep.py"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import torch.distributed as dist

    import bench
    import paper_2604_00785_b200 as b2
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    nccl_id = None
    if world > 1:
        dist.init_process_group("nccl", init_method="env://", device_id=dev)
        ids = [b2.Context.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(ids, src=0)
        nccl_id = ids[0]
    ctx = b2.Context(local, rank=rank, dp=1, ep=world, nccl_id=nccl_id, stream=stream)
    for s in (0.0, 1.0, 1.2):
        for perm in (None, 1):
            if s == 0.0 and perm is not None:
                continue  # uniform: the permutation changes nothing
            r = bench.bench_zipf(torch, b2, ctx, dev, stream, world, rank, s, 10, 3, perm)
            if rank == 0:
                print(json.dumps(r), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
