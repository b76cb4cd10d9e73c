"""World-size-2 gloo tests on CPU of the N > 1 host logic: every rank derives its owned slices
from the C-ABI's shard_slice (optim.cpp:43-50; the EPSO / SO plans of optim.cpp:52-72 use it per
replica group), the slices of a two-member group tile every parameter exactly once, and the
reduce-scatter / all-gather they bound (optim.cpp:148-156, 185-190) reproduce the reference's
member-order fp32 sum bit for bit (two-member sums are exact in any order)."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")

NUMEL = [33, 130_001, 7, 4096, 70_000]  # the optimizer tests' ragged slots


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank(rank, world, port, out):
    import torch.distributed as dist

    import paper_2604_00785_b200 as b2
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ok = True
    for p, n in enumerate(NUMEL):
        b, e = b2.shard_slice(n, world, rank)
        spans = [None] * world
        dist.all_gather_object(spans, (b, e))
        cover = np.zeros(n, np.int32)
        for bb, ee in spans:
            cover[bb:ee] += 1
        ok &= bool((cover == 1).all()) and spans == sorted(spans)
        # reduce-scatter of fp32 grads over the group, then all-gather of the updated slices
        g = torch.from_numpy(np.random.default_rng(100 * p + rank).standard_normal(n).astype(np.float32))
        full = g.clone()
        dist.all_reduce(full)
        parts = [None] * world  # ragged all-gather-v of the owned slices
        dist.all_gather_object(parts, full[b:e].numpy().copy())
        gathered = np.concatenate(parts)
        want = np.zeros(n, np.float32)
        for r in range(world):  # the reference's member-order sum
            want = want + np.random.default_rng(100 * p + r).standard_normal(n).astype(np.float32)
        ok &= bool(np.array_equal(gathered, want))
    flag = torch.tensor([1 if ok else 0])
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    if rank == 0:
        with open(out, "w") as f:
            f.write(str(int(flag.item())))
    dist.destroy_process_group()


def test_two_rank_shard_plan_and_group_sums(tmp_path):
    import torch.multiprocessing as mp
    out = str(tmp_path / "ok.txt")
    for attempt in range(3):  # a free port can be taken before rank 0 binds it
        try:
            mp.spawn(_rank, args=(2, _free_port(), out), nprocs=2, join=True)
            break
        except Exception as exc:  # noqa: BLE001
            if "address already in use" not in str(exc).lower() and "EADDRINUSE" not in str(exc) or attempt == 2:
                raise
    assert open(out).read() == "1"
