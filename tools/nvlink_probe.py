"""NVLink reference point for the EP exchange pattern: NCCL all_to_all_single of 4 x 16,384 x
2048 bf16 rows per rank (every rank sends 1/EP to each peer), timed with CUDA events, max over
ranks — the library collective the owner pulls / pushes of ep_dispatch.cu replace.
    torchrun --nproc-per-node 4 --master-addr 127.0.0.1 tools/nvlink_probe.py"""
import os

import torch
import torch.distributed as dist


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", device_id=dev)
    n = 16384 * 2048 * 4  # bf16 elements per rank (4 layers' token rows: long enough to amortise launch)
    src = torch.randn(n, device=dev).bfloat16()
    dst = torch.empty_like(src)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def timed(fn, iters=20):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        dist.barrier()
        e0.record()
        for _ in range(iters):
            fn()
        e1.record()
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / iters], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    ms = timed(lambda: dist.all_to_all_single(dst, src))
    off_rank = n * 2 * (world - 1) / world  # bytes each rank sends to (and receives from) peers
    if rank == 0:
        print(f"all_to_all_single {n * 2 / 1e6:.0f} MB per rank, EP {world}: {ms:.3f} ms -> "
              f"{off_rank / ms / 1e6:.0f} GB/s per GPU per direction over NVLink")
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
