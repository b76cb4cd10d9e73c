"""Throughput of the sharded-checkpoint record-file path on one GPU.

* GPU crc32 over HBM (b2_crc32) vs the measured HBM peak (a read-only pass) and vs zlib's
  host crc32 (what the reference's crc32_of does, reliability.cpp:58-67) on the same bytes;
* b2_opt_write_shard / b2_opt_restore_shard of an EPSO optimizer holding `--params` elements
  (bf16 weights/grads): bytes / s end to end (gather + crc + D2H + write + fsync), and the
  reader's validate + restore.
Prints one JSON line."""
import argparse
import json
import os
import sys
import tempfile
import time
import zlib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--crc-bytes", type=float, default=4e9)
    ap.add_argument("--params", type=float, default=2.5e8)
    ap.add_argument("--dir", default=None)
    a = ap.parse_args()
    import numpy as np
    import torch

    import paper_2604_00785_b200 as b2
    ctx = b2.Context(0)
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    out = {}
    n = int(a.crc_bytes)
    buf = torch.randint(0, 256, (n,), dtype=torch.uint8, device="cuda")
    b2.crc32(ctx, buf[:1 << 20])
    torch.cuda.synchronize()
    reps = 5
    t0 = time.perf_counter()
    for _ in range(reps):
        c = b2.crc32(ctx, buf)
    dt = (time.perf_counter() - t0) / reps
    out["gpu_crc32"] = {"bytes": n, "s": dt, "GB_s": n / dt / 1e9, "hbm_peak_GB_s": peaks.get("hbm_gbs")}
    host = buf[:1 << 30].cpu().numpy()
    t0 = time.perf_counter()
    hc = zlib.crc32(host)
    hdt = time.perf_counter() - t0
    out["host_zlib_crc32"] = {"bytes": host.size, "s": hdt, "GB_s": host.size / hdt / 1e9, "cores": 1}
    assert b2.crc32(ctx, buf[:1 << 30]) == hc
    del buf
    torch.cuda.empty_cache()

    # a shard of `params` elements: 16 B per element on disk (w16 + master + m + v + g16)
    P = int(a.params)
    sizes = [P // 4, P // 4, P // 4, P - 3 * (P // 4)]
    W = (torch.randn(P, device="cuda") * 0.02).bfloat16()
    G = (torch.randn(P, device="cuda") * 1e-3).bfloat16()
    ps, off = [], 0
    for i, s in enumerate(sizes):
        ps.append((W[off:off + s], G[off:off + s], i % 2, 0))
        off += s
    opt = b2.ShardedOptimizer(ctx, b2.AdamWConfig(warmup_steps=0), ps, b2.EPSO)
    opt.step(stats=False)
    names = [f"p{i}" for i in range(len(sizes))]
    d = a.dir or tempfile.mkdtemp(prefix="ckpt_probe_")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    nbytes, crc, _ = opt.write_shard(d, names)
    wdt = time.perf_counter() - t0
    t0 = time.perf_counter()
    opt.restore_shard(d, names)
    torch.cuda.synchronize()
    rdt = time.perf_counter() - t0
    out["write_shard"] = {"params": P, "file_bytes": nbytes, "s": wdt, "GB_s": nbytes / wdt / 1e9}
    out["restore_shard"] = {"s": rdt, "GB_s_validate_plus_restore": nbytes / rdt / 1e9,
                            "note": "validates the whole file (GPU crc) then reads w16/master/m/v/g16"}
    os.remove(os.path.join(d, "shard-0.bin"))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
