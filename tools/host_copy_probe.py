"""Concurrent pinned host<->device copy bandwidth, one process per GPU (torchrun): what the
e2e leg's per-step copies (x, dout in; out, dx back) can get when every GPU copies at once.
Usage: python -m torch.distributed.run --nproc-per-node N tools/host_copy_probe.py"""
import os

import torch
import torch.distributed as dist


def main():
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    torch.cuda.set_device(rank)
    if world > 1:
        dist.init_process_group("gloo")
    n = 64 << 20  # 64 MiB = one [16384, 2048] bf16 tensor
    h_in = [torch.empty(n, dtype=torch.uint8).pin_memory() for _ in range(2)]
    h_out = [torch.empty(n, dtype=torch.uint8).pin_memory() for _ in range(2)]
    d = [torch.empty(n, dtype=torch.uint8, device="cuda") for _ in range(4)]
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
    for label, both in (("H2D only", False), ("H2D + D2H concurrently", True)):
        for it in range(2):
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10):
                with torch.cuda.stream(s_in):
                    for k in range(2):
                        d[k].copy_(h_in[k], non_blocking=True)
                if both:
                    with torch.cuda.stream(s_out):
                        for k in range(2):
                            h_out[k].copy_(d[2 + k], non_blocking=True)
            torch.cuda.current_stream().wait_stream(s_in)
            torch.cuda.current_stream().wait_stream(s_out)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 10
        gbs = 2 * n / (ms * 1e-3) / 1e9
        print(f"rank {rank}/{world}: {label}: {ms:.2f} ms per 128 MiB each way -> {gbs:.1f} GB/s per direction",
              flush=True)


if __name__ == "__main__":
    main()
