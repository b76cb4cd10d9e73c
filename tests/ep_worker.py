"""Multi-GPU worker for the expert-parallel parity tests (one process per GPU).

Each rank runs the B200 MoE layer on its S-token slice with its N/EP experts
(dispatch/combine over NVLink peer memory); rank 0 gathers every rank's outputs and
gradients and compares them with the oracle's EP world (oracle/moe_oracle.c, itself
pinned bitwise to the reference's fast_moe_forward/backward at EP > 1).
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def rel_err(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b) / np.maximum(1.0, np.maximum(np.abs(a), np.abs(b))))) if a.size else 0.0


def scale_err(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-30)) if a.size else 0.0


def run(rank, world, port, case, result_path):
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
    c = dict(case)
    ckpt, graph, no_overlap = c.pop("ckpt", False), c.pop("graph", False), c.pop("no_overlap", False)
    stream = torch.cuda.Stream() if graph else None  # graph capture needs a non-default stream
    if stream is not None:
        torch.cuda.set_stream(stream)
    ctx = b2.Context(rank, rank=rank, dp=1, ep=world, nccl_id=ids[0], stream=stream)

    s = c.pop("s")
    dtype = torch.float32 if c.pop("dtype") == "f32" else torch.bfloat16
    fur = c.pop("fur", False)
    c["ep"] = world
    ocfg, bcfg = bind.moe_cfg(**c), b2.MoeConfig(**c)
    orc = bind.get("orc")
    H, N, I, K = ocfg.hidden, ocfg.n_experts, ocfg.intermediate, ocfg.top_k
    NR = N // world
    std = 0.2 if dtype == torch.float32 else 0.02
    router, gate, up, down = orc.expert_weights(ocfg, 1234, std)
    x = orc.normal((world * s, H), 77, 0, 0.7 if dtype == torch.float32 else 1.0)
    dout = orc.normal((world * s, H), 78, 0, 1.0)
    if dtype == torch.bfloat16:
        rb = lambda a: torch.from_numpy(np.ascontiguousarray(a)).bfloat16().float().numpy()
        router, gate, up, down, x, dout = map(rb, (router, gate, up, down, x, dout))
    dev = torch.device("cuda", rank)
    tt = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev).to(dtype)
    sl = slice(rank * s, (rank + 1) * s)
    el = slice(rank * NR, (rank + 1) * NR)
    X, DO = tt(x[sl]), tt(dout[sl])
    R, G, U, D = tt(router), tt(gate[el]), tt(up[el]), tt(down[el])
    layer = b2.MoeLayer(ctx, bcfg, dtype, s, checkpoint=ckpt)
    if no_overlap:  # dX return after the weight-gradient GEMMs (the fp32 path's order)
        import ctypes
        b2.lib().b2x_moe_set_overlap_return.argtypes = [ctypes.c_void_p, ctypes.c_int]
        assert b2.lib().b2x_moe_set_overlap_return(layer.h, 0) == 0
    reps = 3 if graph else 1  # eager, capture, replay: the last one is checked
    if graph:
        layer.set_graph(True)
    out, apg = torch.empty_like(X), torch.empty((s, N), dtype=torch.float32, device=dev)
    g = dict(input=torch.empty_like(X), router=torch.empty_like(R), gate=torch.empty_like(G), up=torch.empty_like(U),
             down=torch.empty_like(D))
    for _ in range(reps):
        layer.forward(X, R, G, U, D, fur=fur, out=out)
        layer.aux_probs_grad(0.01, out=apg)
        layer.backward(R, G, U, D, DO, apg, grads=g)
    torch.cuda.synchronize()
    mine = {
        "out": out.float().cpu(), "dx": g["input"].float().cpu(), "drouter": g["router"].float().cpu(),
        "dgate": g["gate"].float().cpu(), "dup": g["up"].float().cpu(), "ddown": g["down"].float().cpu(),
        "aux": torch.tensor([layer.aux_loss()], dtype=torch.float64),
    }
    art = layer.artifacts()
    gathered = [None] * world
    dist.all_gather_object(gathered, {"t": mine, "art": art})
    if rank == 0:
        ref = orc.moe_layer(ocfg, s, x, router, gate, up, down, dout, fur=fur, aux_coeff=0.01)
        cat = lambda key: np.concatenate([gathered[r]["t"][key].numpy() for r in range(world)])
        res = {}
        if dtype == torch.float32:
            res["out"] = rel_err(cat("out"), ref["out"])
            res["dx"] = rel_err(cat("dx"), ref["dx"])
            res["dgate"] = rel_err(cat("dgate"), ref["dgate"])
            res["dup"] = rel_err(cat("dup"), ref["dup"])
            res["ddown"] = rel_err(cat("ddown"), ref["ddown"])
            res["drouter"] = max(rel_err(gathered[r]["t"]["drouter"].numpy(), ref["drouter"][r]) for r in range(world))
        else:
            res["out"] = rel_err(cat("out"), ref["out"])
            res["dx"] = rel_err(cat("dx"), ref["dx"])
            res["dgate"] = scale_err(cat("dgate"), ref["dgate"])
            res["dup"] = scale_err(cat("dup"), ref["dup"])
            res["ddown"] = scale_err(cat("ddown"), ref["ddown"])
            res["drouter"] = max(scale_err(gathered[r]["t"]["drouter"].numpy(), ref["drouter"][r]) for r in range(world))
        res["aux"] = max(abs(float(gathered[r]["t"]["aux"][0]) - ref["aux"][r]) for r in range(world))
        # integer artifacts bit-exact against the oracle's per-rank count_tokens/generate_indices
        table = ref["indices"] if not fur else (
            (np.arange(world * s)[:, None] % s * K + np.arange(K)[None, :]) % N)
        bad = []
        for r in range(world):
            want = orc.artifacts(ocfg, table.astype(np.int64), r)
            got = gathered[r]["art"]
            for key in ("token_counts", "partial_token_counts", "partial_cum", "cum_token_counts", "expert_counts",
                        "cum_expert_counts", "input_indices", "output_indices", "selected_k", "counter"):
                if not np.array_equal(np.asarray(got[key]).reshape(-1), np.asarray(want[key]).reshape(-1)):
                    bad.append(f"rank{r}:{key}")
        res["artifacts_mismatch"] = bad
        with open(result_path, "w") as f:
            import json
            json.dump(res, f)
    dist.barrier()
    layer.close()
    ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    import json
    rank, world, port = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
    case = json.loads(sys.argv[4])
    run(rank, world, port, case, sys.argv[5])
