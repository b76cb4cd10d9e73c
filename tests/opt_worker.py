"""Multi-GPU worker for the sharded-optimizer parity tests (one process per GPU).

Every rank steps b2.ShardedOptimizer (NCCL reduce-scatter / all-gather over the DP,
EP and DP x EP communicators) on its own synthetic gradients; rank 0 compares every
rank's final weights, fp32 masters, moments and step statistics with the oracle's
ShardedOptimizer world (oracle/moe_oracle.c, pinned bitwise to optim.cpp:109-194).
fp32 grads keep NCCL's sums of two members exact, so 2-member groups are bitwise.
bf16=1: the benchmarked path — bf16 weights and grads on the GPU (NCCL reduce-scatters the bf16
grads) against the oracle's fp32 sums of the same bf16-rounded values (optim.cpp:148-156).
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

NUMEL = [33, 30, 7, 1029]
CLS = [0, 1, 0, 1]


def run(rank, world, port, dp, ep, mode, result_path, bf16=False):
    import torch
    import torch.distributed as dist

    import paper_2604_00785_b200 as b2
    from oracle import bind

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(rank)
    ids = [b2.Context.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(ids, src=0)
    ctx = b2.Context(rank, rank=rank, dp=dp, ep=ep, nccl_id=ids[0])
    orc = bind.get("orc")
    total = sum(NUMEL)
    steps = 6
    rng = np.random.default_rng(1000 + dp * 10 + ep + mode)
    w0 = np.zeros((world, total), np.float32)
    for r in range(world):
        e = r % ep
        off = 0
        for p, (n, c) in enumerate(zip(NUMEL, CLS)):
            w0[r, off:off + n] = orc.normal((n,), 402 + p, 100 + e if c else 1, 0.05)
            off += n
    grads = (rng.standard_normal((steps, world, total)) * 0.5).astype(np.float32)
    wdt = torch.bfloat16 if bf16 else torch.float32
    if bf16:  # both sides see the same bf16 values
        rb = lambda a: torch.from_numpy(a).bfloat16().float().numpy()
        w0, grads = rb(w0), rb(grads)
    cfg = b2.AdamWConfig(warmup_steps=2, total_steps=100, peak_lr=1e-2, min_lr=1e-3)
    dev = torch.device("cuda", rank)
    W = torch.from_numpy(w0[rank].copy()).to(dev).to(wdt)
    G = torch.zeros(total, dtype=wdt, device=dev)
    params, off = [], 0
    for n, c in zip(NUMEL, CLS):
        params.append((W[off:off + n], G[off:off + n], c, 0))
        off += n
    opt = b2.ShardedOptimizer(ctx, cfg, params, mode)
    stats = []
    for s in range(steps):
        G.copy_(torch.from_numpy(grads[s, rank]).to(wdt))
        st = opt.step(stats=True)
        stats.append([st["lr"], st["grad_norm"], st["clip_scale"]])
    torch.cuda.synchronize()
    # checkpoint assembly: every member's full state must equal the members' owned slices
    # stitched together (each rank checks its own view against the oracle's per-rank slices)
    full = [opt.gather_state(p, n) for p, n in enumerate(NUMEL)]
    mine = {"w": W.float().cpu().numpy().tolist(), "stats": stats, "sb": opt.state_bytes(),
            "full_master": [f[0].tolist() for f in full], "owned": [list(opt.owned(p)) for p in range(len(NUMEL))],
            "master": [opt.state(p)[0].tolist() for p in range(len(NUMEL))],
            "m": [opt.state(p)[1].tolist() for p in range(len(NUMEL))],
            "v": [opt.state(p)[2].tolist() for p in range(len(NUMEL))]}
    # record-file checkpoint round trip (reliability.cpp:402-460 / 623-675): write the shard
    # files, restore into a fresh optimizer, then one more identical step on both
    ck = os.path.join(os.path.dirname(result_path), "ckpt")
    if bf16:  # the shard-file round trip is covered by the fp32 runs
        return finish(rank, world, dp, ep, mode, result_path, orc, mine, grads, w0, opt, ctx, dist, bf16)
    if rank == 0:
        os.makedirs(ck, exist_ok=True)
    dist.barrier()
    names = [f"layer.p{p}" for p in range(len(NUMEL))]
    nbytes, _, shard = opt.write_shard(ck, names)
    torch.cuda.synchronize()
    # the .g16 records hold the WRITER's grads (reliability.cpp:455): expert params come from
    # this rank's model-shard file, non-expert params from the ep-0 shard (restore_full)
    writers = [None] * world
    dist.all_gather_object(writers, (shard, nbytes > 0, G.cpu().numpy()))
    g_of = {sh: g for sh, w, g in writers if w}
    g_exp = np.empty(total, np.float32)
    off = 0
    for n, c in zip(NUMEL, CLS):
        src = g_of[shard] if c else g_of[min(g_of)]
        g_exp[off:off + n] = src[off:off + n]
        off += n
    g_exp = torch.from_numpy(g_exp).to(dev).bfloat16().float()
    dist.barrier()
    W2 = torch.zeros_like(W)
    G2 = torch.zeros_like(G)
    params2, off = [], 0
    for n, c in zip(NUMEL, CLS):
        params2.append((W2[off:off + n], G2[off:off + n], c, 0))
        off += n
    opt2 = b2.ShardedOptimizer(ctx, cfg, params2, mode)
    opt2.restore_shard(ck, names)
    opt2.set_step_count(steps)
    torch.cuda.synchronize()
    same_state = lambda: all(np.array_equal(a, b_) for p in range(len(NUMEL)) for a, b_ in zip(opt.state(p), opt2.state(p)))
    detail = {"w": bool(torch.equal(W2, W)), "g": bool(torch.equal(G2, g_exp)), "state": same_state()}
    G.copy_(G2)
    opt.step(stats=False)
    opt2.step(stats=False)
    torch.cuda.synchronize()
    detail["w_after"] = bool(torch.equal(W2, W))
    detail["state_after"] = same_state()
    if nbytes:  # the writer's file parses under the oracle's read_record_file
        cnt, _ = orc.record_file_read(os.path.join(ck, f"shard-{shard}.bin"))
        detail["file"] = cnt > 0 and nbytes == os.path.getsize(os.path.join(ck, f"shard-{shard}.bin"))
    mine["ckpt_ok"] = all(detail.values())
    mine["ckpt_detail"] = detail
    opt2.close()
    return finish(rank, world, dp, ep, mode, result_path, orc, mine, grads, w0, opt, ctx, dist, bf16)


def finish(rank, world, dp, ep, mode, result_path, orc, mine, grads, w0, opt, ctx, dist, bf16):
    mine.setdefault("ckpt_ok", True)
    mine.setdefault("ckpt_detail", {})
    gathered = [None] * world
    dist.all_gather_object(gathered, mine)
    if rank == 0:
        ocfg = orc.adamw_cfg(warmup_steps=2, total_steps=100, peak_lr=1e-2, min_lr=1e-3)
        ref = orc.sharded_steps(dp, ep, 1, mode, ocfg, NUMEL, CLS, [0] * len(NUMEL), w0, grads)
        res = {"weights_equal": True, "state_equal": True, "stats_maxdiff": 0.0, "state_bytes_equal": True,
               "weights_maxrel": 0.0, "state_maxrel": 0.0}
        for r in range(world):
            g = gathered[r]
            wg = np.asarray(g["w"], np.float32)
            if not np.array_equal(wg, ref["weights"][r]):
                res["weights_equal"] = False
            d = np.abs(wg.astype(np.float64) - ref["weights"][r]) / np.maximum(1.0, np.abs(ref["weights"][r]))
            res["weights_maxrel"] = max(res["weights_maxrel"], float(d.max()))
            packed = [np.concatenate([np.asarray(g[k][p], np.float32) for p in range(len(NUMEL))]) for k in
                      ("master", "m", "v")]
            n_own = packed[0].size
            for arr, key in zip(packed, ("master", "m", "v")):
                want = ref[key][r][:n_own]
                if not np.array_equal(arr, want):
                    res["state_equal"] = False
                d = np.abs(arr.astype(np.float64) - want) / np.maximum(1.0, np.abs(want))
                res["state_maxrel"] = max(res["state_maxrel"], float(d.max()) if d.size else 0.0)
            res["stats_maxdiff"] = max(res["stats_maxdiff"],
                                       float(np.max(np.abs(np.asarray(g["stats"]) - ref["stats"][:, r, :]))))
            if g["sb"] != int(ref["state_bytes"][r]):
                res["state_bytes_equal"] = False
        # gathered full masters: rank r's full view of param p must hold, on every slice owned
        # by a member q of r's owning group, exactly q's owned master
        res["gather_ok"] = True
        for p in range(len(NUMEL)):
            for r in range(world):
                got = np.asarray(gathered[r]["full_master"][p], np.float32)
                for q in range(world):
                    same_ep = (r % ep) == (q % ep)
                    if mode == 0:
                        members = q == r
                    elif mode == 2 and CLS[p] == 0:
                        members = True  # EPSO non-expert: the fused DP x EP group
                    else:
                        members = same_ep  # expert params, and SO: the EP-orthogonal DP group
                    if not members:
                        continue
                    b_, e_ = gathered[q]["owned"][p]
                    if not np.array_equal(got[b_:e_], np.asarray(gathered[q]["master"][p], np.float32)):
                        res["gather_ok"] = False
        res["ckpt_ok"] = all(g["ckpt_ok"] for g in gathered)
        res["ckpt_detail"] = [g["ckpt_detail"] for g in gathered]
        with open(result_path, "w") as f:
            json.dump(res, f)
    dist.barrier()
    opt.close()
    ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    rank, world, port = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
    dp, ep, mode = int(sys.argv[4]), int(sys.argv[5]), int(sys.argv[6])
    run(rank, world, port, dp, ep, mode, sys.argv[7], len(sys.argv) > 8 and sys.argv[8] == "1")
