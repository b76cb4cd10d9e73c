"""Parity of the CUDA MoE path (through the C-ABI) with the CPU oracle.

Bars (BASELINE.json north star, metric of tests/test_util.hpp:15-18
rel_err = |a-b| / max(1,|a|,|b|)):
  * routing top-k indices and the permutation: bit-exact given identical scores;
  * fp32 mode: every output / gradient within 1e-4 rel_err of the fp32 oracle;
  * bf16 mode vs the fp32 oracle on the same bf16-rounded inputs: outputs and input
    grads within 2e-2 rel_err elementwise; weight / router grads within 2e-2 of
    the tensor scale (max|d| / max|ref|: long bf16 reductions cancel).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import bind

pytestmark = pytest.mark.gpu

TOL_F32 = 1e-4
TOL_BF16 = 2e-2


def rel_err(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b) / np.maximum(1.0, np.maximum(np.abs(a), np.abs(b))))) if a.size else 0.0


def scale_err(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-30)) if a.size else 0.0


@pytest.fixture(scope="module")
def b2ctx():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2604_00785_b200 as b2
    return b2, b2.Context(0)


def cfg_pair(**kw):
    import paper_2604_00785_b200 as b2
    return bind.moe_cfg(**kw), b2.MoeConfig(**kw)


# ---------------------------------------------------------------- routing

@pytest.mark.parametrize("n,k,normalize", [(8, 2, False), (64, 8, False), (12, 3, True), (96, 8, False)])
def test_softmax_topk_bit_exact_on_identical_scores(b2ctx, orc, n, k, normalize):
    b2, ctx = b2ctx
    rng = np.random.default_rng(n * 7 + k)
    logits = rng.standard_normal((777, n)).astype(np.float32)
    logits[::5, 3] = logits[::5, 1]  # exact ties -> lower index
    logits[::7, : n // 2] = 0.0
    probs_o, w_o, i_o = orc.softmax_topk(logits, k)
    if normalize:
        w_o = w_o / w_o.sum(1, keepdims=True, dtype=np.float32)
    probs, w, idx = b2.softmax_topk(ctx, torch.from_numpy(logits).cuda(), k, normalize)
    assert np.array_equal(idx.cpu().numpy(), i_o)
    assert np.array_equal(probs.cpu().numpy(), probs_o)
    if not normalize:
        assert np.array_equal(w.cpu().numpy(), w_o)
    else:
        assert rel_err(w.cpu().numpy(), w_o) <= 1e-6


@pytest.mark.parametrize("H,N,K", [(32, 8, 2), (256, 64, 8)])
def test_route_logits_bitwise(b2ctx, orc, H, N, K):
    b2, ctx = b2ctx
    ocfg, bcfg = cfg_pair(n_experts=N, top_k=K, hidden=H, intermediate=64)
    x = orc.normal((300, H), 77, 0, 1.0)
    router = orc.normal((H, N), 5, 1, 0.2)
    lo, po, wo, io = orc.route_f32(ocfg, x, router)
    logits, probs, w, idx = b2.route(ctx, bcfg, torch.from_numpy(x).cuda(), torch.from_numpy(router).cuda())
    assert np.array_equal(logits.cpu().numpy(), lo)
    assert np.array_equal(idx.cpu().numpy(), io)
    assert np.array_equal(w.cpu().numpy(), wo)


@pytest.mark.parametrize("S,H,N,K", [(300, 2048, 64, 8), (129, 256, 96, 8), (64, 64, 8, 2), (77, 96, 24, 3),
                                     (1000, 160, 200, 4)])
def test_route_logits_bf16_bitwise(b2ctx, orc, S, H, N, K):
    """bf16 inputs take the cp.async/f32x2 logits kernel (H % 32 == 0, N % 8 == 0):
    bit-identical to the reference's fp32 multiply-then-add on the same rounded values."""
    b2, ctx = b2ctx
    ocfg, bcfg = cfg_pair(n_experts=N, top_k=K, hidden=H, intermediate=64)
    rb = lambda a: torch.from_numpy(np.ascontiguousarray(a)).bfloat16()
    x, router = rb(orc.normal((S, H), 77, 0, 1.0)), rb(orc.normal((H, N), 5, 1, 0.2))
    lo, po, wo, io = orc.route_f32(ocfg, x.float().numpy(), router.float().numpy())
    logits, probs, w, idx = b2.route(ctx, bcfg, x.cuda(), router.cuda())
    assert np.array_equal(logits.cpu().numpy(), lo)
    assert np.array_equal(idx.cpu().numpy(), io)
    assert np.array_equal(w.cpu().numpy(), wo)


FOUR = np.array([[0, 1], [0, 2], [1, 3], [2, 3]], np.int64)


def _compare_artifacts(got, want):
    for key in ("token_counts", "partial_token_counts", "partial_cum", "cum_token_counts", "expert_counts",
                "cum_expert_counts", "input_indices", "output_indices", "selected_k", "counter"):
        assert np.array_equal(np.asarray(got[key]), np.asarray(want[key])), key
    assert got["rt"] == want["rt"] and got["th"] == want["th"]


def test_artifacts_four_token_example(b2ctx, orc):
    b2, ctx = b2ctx
    ocfg, bcfg = cfg_pair(n_experts=4, top_k=2, hidden=4, intermediate=4, ep=2, token_block=8)
    t = torch.from_numpy(FOUR.astype(np.int32)).cuda()
    a = b2.routing_artifacts(ctx, bcfg, t, 0)
    assert a["input_indices"].tolist() == [0, 1, 0, 2]  # test_moe.cpp:110-119
    assert a["output_indices"].tolist() == [0, 2, 1, 3]
    assert a["selected_k"].tolist() == [0, 1, 0, 0]
    for r in (0, 1):
        _compare_artifacts(b2.routing_artifacts(ctx, bcfg, t, r), orc.artifacts(ocfg, FOUR, r))


def test_artifacts_out_of_range_raises(b2ctx):
    b2, ctx = b2ctx
    _, bcfg = cfg_pair(n_experts=4, top_k=2, hidden=4, intermediate=4, ep=2)
    t = torch.tensor([[0, 1], [2, 7]], dtype=torch.int32, device="cuda")
    with pytest.raises(b2.ContractError):
        b2.routing_artifacts(ctx, bcfg, t, 0)


@pytest.mark.parametrize("seed", range(12))
def test_artifacts_random_tables_bit_exact(b2ctx, orc, seed):
    b2, ctx = b2ctx
    rng = np.random.default_rng(seed)
    ep = int(rng.integers(1, 5))
    n = ep * int(rng.integers(1, 17))
    k = int(rng.integers(1, min(8, n) + 1))
    T = int(rng.integers(1, 3000)) if seed % 3 else int(rng.integers(1, 40))
    if seed % 2:  # distinct experts per token, like a real top-k
        idx = np.stack([rng.permutation(n)[:k] for _ in range(T)]).astype(np.int64)
    else:  # repeated experts allowed (test_moe.cpp:84-103)
        idx = rng.integers(0, n, size=(T, k)).astype(np.int64)
    kw = dict(n_experts=n, top_k=k, hidden=8, intermediate=8, ep=ep, token_block=int(rng.integers(1, 9)))
    ocfg, bcfg = cfg_pair(**kw)
    t = torch.from_numpy(idx.astype(np.int32)).cuda()
    for r in range(ep):
        _compare_artifacts(b2.routing_artifacts(ctx, bcfg, t, r), orc.artifacts(ocfg, idx, r))


# ---------------------------------------------------------------- full layer

def run_layer(b2, ctx, bcfg, dtype, x, router, gate, up, down, dout, fur=False, aux_coeff=0.0):
    tt = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda().to(dtype)
    X, R, G, U, D, DO = map(tt, (x, router, gate, up, down, dout))
    layer = b2.MoeLayer(ctx, bcfg, dtype, x.shape[0])
    out = layer.forward(X, R, G, U, D, fur=fur)
    apg = layer.aux_probs_grad(aux_coeff) if aux_coeff else None
    grads = layer.backward(R, G, U, D, DO, apg)
    torch.cuda.synchronize()
    res = {k: v.float().cpu().numpy() for k, v in grads.items()}
    res["out"] = out.float().cpu().numpy()
    res["probs"], res["weights"], res["indices"] = layer.routing()
    res["artifacts"] = layer.artifacts()
    res["aux"] = layer.aux_loss()
    res["launches"] = layer.last_launches()
    return res


F32_CASES = [
    dict(n_experts=8, top_k=2, hidden=32, intermediate=48, token_block=8, s=64),
    dict(n_experts=6, top_k=3, hidden=20, intermediate=12, token_block=3, s=37, normalize_topk=True),
    dict(n_experts=8, top_k=2, hidden=16, intermediate=24, token_block=4, s=16, fur=True),
    dict(n_experts=64, top_k=8, hidden=128, intermediate=64, token_block=8, s=256),
    dict(n_experts=1, top_k=1, hidden=5, intermediate=7, token_block=8, s=6),
    # top_k > 32: the router backward's serial per-k path (router_dlogits_kernel)
    dict(n_experts=40, top_k=34, hidden=16, intermediate=8, token_block=4, s=24, normalize_topk=True),
]


@pytest.mark.parametrize("case", F32_CASES, ids=lambda c: f"n{c['n_experts']}k{c['top_k']}h{c['hidden']}")
def test_layer_fp32_matches_oracle(b2ctx, orc, case):
    b2, ctx = b2ctx
    c = dict(case)
    s = c.pop("s")
    fur = c.pop("fur", False)
    ocfg, bcfg = cfg_pair(**c)
    router, gate, up, down = orc.expert_weights(ocfg, 1234, 0.2)
    x = orc.normal((s, ocfg.hidden), 77, 0, 0.7)
    dout = orc.normal((s, ocfg.hidden), 78, 0, 1.0)
    ref = orc.moe_layer(ocfg, s, x, router, gate, up, down, dout, fur=fur, aux_coeff=0.01)
    got = run_layer(b2, ctx, bcfg, torch.float32, x, router, gate, up, down, dout, fur=fur, aux_coeff=0.01)
    assert np.array_equal(got["indices"], ref["indices"])
    assert np.array_equal(got["weights"], ref["weights"])
    assert rel_err(got["aux"], ref["aux"][0]) <= TOL_F32
    if fur:  # fur_route (moe.hpp:84-99) replaces the dispatch table
        table = (np.arange(s)[:, None] * ocfg.top_k + np.arange(ocfg.top_k)[None, :]) % ocfg.n_experts
    else:
        table = ref["indices"]
    art_ref = orc.artifacts(ocfg, table.astype(np.int64), 0)
    _compare_artifacts(got["artifacts"], art_ref)
    for key, gkey in [("out", "out"), ("dx", "input"), ("drouter", "router"), ("dgate", "gate"), ("dup", "up"),
                      ("ddown", "down")]:
        want = ref[key][0] if key == "drouter" else ref[key]
        e = rel_err(got[gkey], want)
        assert e <= TOL_F32, f"{key}: rel_err {e}"
    assert got["launches"] > 0


BF16_CASES = [
    dict(n_experts=8, top_k=2, hidden=256, intermediate=256, s=512),
    dict(n_experts=64, top_k=8, hidden=256, intermediate=128, s=512),
    dict(n_experts=16, top_k=4, hidden=384, intermediate=192, s=333),
]


@pytest.mark.parametrize("case", BF16_CASES, ids=lambda c: f"n{c['n_experts']}k{c['top_k']}h{c['hidden']}")
def test_layer_bf16_matches_fp32_oracle(b2ctx, orc, case):
    b2, ctx = b2ctx
    c = dict(case)
    s = c.pop("s")
    ocfg, bcfg = cfg_pair(**c)
    rb = lambda a: torch.from_numpy(np.ascontiguousarray(a)).bfloat16().float().numpy()
    router, gate, up, down = (rb(t) for t in orc.expert_weights(ocfg, 1234, 0.02))
    x = rb(orc.normal((s, ocfg.hidden), 77, 0, 1.0))
    dout = rb(orc.normal((s, ocfg.hidden), 78, 0, 1.0))
    ref = orc.moe_layer(ocfg, s, x, router, gate, up, down, dout, aux_coeff=0.01)
    got = run_layer(b2, ctx, bcfg, torch.bfloat16, x, router, gate, up, down, dout, aux_coeff=0.01)
    # identical fp32 router math on identical inputs -> identical routing
    assert np.array_equal(got["indices"], ref["indices"])
    _compare_artifacts(got["artifacts"], orc.artifacts(ocfg, ref["indices"], 0))
    assert rel_err(got["out"], ref["out"]) <= TOL_BF16
    assert rel_err(got["input"], ref["dx"]) <= TOL_BF16
    for key, gkey in [("drouter", "router"), ("dgate", "gate"), ("dup", "up"), ("ddown", "down")]:
        want = ref[key][0] if key == "drouter" else ref[key]
        e = scale_err(got[gkey], want)
        assert e <= TOL_BF16, f"{key}: scale_err {e}"


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_graph_replay_matches_eager(b2ctx, dtype):
    """CUDA-graph mode: the captured forward/backward replays bit-identically to the
    eager path, including after the inputs behind the same pointers change (every
    data-dependent size is read on the device)."""
    b2, _ = b2ctx
    dt = torch.bfloat16 if dtype == "bf16" else torch.float32
    stream = torch.cuda.Stream()
    ctx = b2.Context(0, stream=stream)
    cfg = b2.MoeConfig(n_experts=16, top_k=4, hidden=256, intermediate=128)
    S = 300
    gen = torch.Generator(device="cuda").manual_seed(5)
    mk = lambda shape, std: (torch.randn(shape, device="cuda", generator=gen) * std).to(dt)
    router, gate, up, down = mk((256, 16), 0.05), mk((16, 256, 128), 0.05), mk((16, 256, 128), 0.05), \
        mk((16, 128, 256), 0.05)
    xs = [mk((S, 256), 1.0) for _ in range(3)]
    douts = [mk((S, 256), 1.0) for _ in range(3)]

    def run(layer, x_buf, d_buf, out, apg, grads, i):
        with torch.cuda.stream(stream):
            x_buf.copy_(xs[i])
            d_buf.copy_(douts[i])
            layer.forward(x_buf, router, gate, up, down, out=out)
            layer.aux_probs_grad(0.01, out=apg)
            layer.backward(router, gate, up, down, d_buf, apg, grads=grads)
        stream.synchronize()
        return [out.clone()] + [grads[k].clone() for k in ("input", "router", "gate", "up", "down")]

    def bufs():
        with torch.cuda.stream(stream):
            out = torch.empty((S, 256), dtype=dt, device="cuda")
            grads = dict(input=torch.empty((S, 256), dtype=dt, device="cuda"), router=torch.empty_like(router),
                         gate=torch.empty_like(gate), up=torch.empty_like(up), down=torch.empty_like(down))
            apg = torch.empty((S, 16), dtype=torch.float32, device="cuda")
            return torch.empty_like(xs[0]), torch.empty_like(douts[0]), out, apg, grads

    eager = b2.MoeLayer(ctx, cfg, dt, S)
    want = [run(eager, *bufs(), i) for i in range(3)]
    graphed = b2.MoeLayer(ctx, cfg, dt, S)
    graphed.set_graph(True)
    b = bufs()
    got = [run(graphed, *b, i) for i in (0, 1, 2, 0, 1)]  # eager, capture, replay x3
    for g, i in zip(got, (0, 1, 2, 0, 1)):
        for a, w in zip(g, want[i]):
            assert torch.equal(a, w)
    assert graphed.last_launches() > 0
    # in-graph stage profiling (mode 2): event-record nodes around every stage of the captured
    # graphs; the replays stay bitwise equal and every stage reports a positive time
    graphed.set_profiling(2)
    got = [run(graphed, *b, i) for i in (0, 1, 2)]  # eager, capture (with the events), replay
    for g, i in zip(got, (0, 1, 2)):
        for a, w in zip(g, want[i]):
            assert torch.equal(a, w)
    st = graphed.stage_times()
    assert all(v > 0 for k, v in st.items() if k.startswith("gemm")), st
    graphed.set_profiling(False)


def zipf_inputs(S, H, N, s, seed=4242):
    """Config-E style skewed routing: logits[t,e] = log z_e + Gumbel(t,e) with
    z_e ∝ (e+1)^-s (identity permutation: the hottest experts first). Realised through the
    layer's own router: x[t, :N] holds the logits, Wr = [I_N; 0], so x·Wr reproduces them."""
    rng = np.random.default_rng(seed)
    z = (np.arange(N) + 1.0) ** -s
    z /= z.sum()
    gumbel = -np.log(-np.log(rng.uniform(1e-12, 1.0, (S, N))))
    x = rng.standard_normal((S, H)).astype(np.float32)
    x[:, :N] = (np.log(z)[None, :] + gumbel).astype(np.float32)
    router = np.zeros((H, N), np.float32)
    router[np.arange(N), np.arange(N)] = 1.0
    return x, router


@pytest.mark.parametrize("s,K", [(1.2, 4), (3.0, 1)])
def test_layer_bf16_zipf_skewed_routing(b2ctx, orc, s, K):
    """Load-imbalance stress: hot experts get many 256-row tiles, cold ones few or none
    (empty groups in every GEMM kind, zero weight-gradients)."""
    b2, ctx = b2ctx
    S, H, N, I = 512, 256, 16, 128
    ocfg, bcfg = cfg_pair(n_experts=N, top_k=K, hidden=H, intermediate=I)
    rb = lambda a: torch.from_numpy(np.ascontiguousarray(a)).bfloat16().float().numpy()
    x, router = zipf_inputs(S, H, N, s)
    x, router = rb(x), rb(router)
    _, gate, up, down = (rb(t) for t in orc.expert_weights(ocfg, 1234, 0.02))
    dout = rb(orc.normal((S, H), 78, 0, 1.0))
    ref = orc.moe_layer(ocfg, S, x, router, gate, up, down, dout, aux_coeff=0.01)
    counts = np.bincount(ref["indices"].ravel(), minlength=N)
    assert counts.max() >= 3 * counts.mean() and (s < 2 or counts.min() == 0), counts
    got = run_layer(b2, ctx, bcfg, torch.bfloat16, x, router, gate, up, down, dout, aux_coeff=0.01)
    assert np.array_equal(got["indices"], ref["indices"])
    _compare_artifacts(got["artifacts"], orc.artifacts(ocfg, ref["indices"], 0))
    assert rel_err(got["out"], ref["out"]) <= TOL_BF16
    assert rel_err(got["input"], ref["dx"]) <= TOL_BF16
    for key, gkey in [("drouter", "router"), ("dgate", "gate"), ("dup", "up"), ("ddown", "down")]:
        want = ref[key][0] if key == "drouter" else ref[key]
        e = scale_err(got[gkey], want)
        assert e <= TOL_BF16, f"{key}: scale_err {e}"
    # experts that received no rows have exactly zero weight gradients
    for e in np.where(counts == 0)[0]:
        assert not got["gate"][e].any() and not got["up"][e].any() and not got["down"][e].any()


def test_host_pipeline_matches_synchronous(b2ctx):
    """b2_moe_fwd_bwd_host_async (two staging slots, copies overlapped with compute) gives
    every step exactly the results of the synchronous host-buffer call."""
    b2, _ = b2ctx
    stream = torch.cuda.Stream()
    ctx = b2.Context(0, stream=stream)
    cfg = b2.MoeConfig(n_experts=16, top_k=4, hidden=256, intermediate=128)
    S = 256
    gen = torch.Generator(device="cuda").manual_seed(21)
    mk = lambda shape, std: (torch.randn(shape, device="cuda", generator=gen) * std).bfloat16()
    router, gate, up, down = mk((256, 16), 0.05), mk((16, 256, 128), 0.05), mk((16, 256, 128), 0.05), \
        mk((16, 128, 256), 0.05)
    xs = [mk((S, 256), 1.0).cpu().pin_memory() for _ in range(4)]
    ds = [mk((S, 256), 1.0).cpu().pin_memory() for _ in range(4)]
    grads = lambda: dict(router=torch.empty_like(router), gate=torch.empty_like(gate), up=torch.empty_like(up),
                         down=torch.empty_like(down))
    ref_layer, pipe_layer = b2.MoeLayer(ctx, cfg, torch.bfloat16, S), b2.MoeLayer(ctx, cfg, torch.bfloat16, S)
    pipe_layer.set_graph(True)
    want, outs = [], []
    for i in range(4):
        o, d, g = torch.empty_like(xs[i]).pin_memory(), torch.empty_like(xs[i]).pin_memory(), grads()
        ref_layer.fwd_bwd_host(xs[i], ds[i], router, gate, up, down, o, d, g, 0.01)
        want.append((o, d))
    g = grads()
    for i in range(4):
        o, d = torch.empty_like(xs[i]).pin_memory(), torch.empty_like(xs[i]).pin_memory()
        pipe_layer.fwd_bwd_host(xs[i], ds[i], router, gate, up, down, o, d, g, 0.01, wait=False)
        outs.append((o, d))
    pipe_layer.host_wait()
    for (o, d), (wo, wd) in zip(outs, want):
        assert torch.equal(o, wo) and torch.equal(d, wd)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_checkpoint_replay_bitwise_and_lighter(b2ctx, dtype):
    """moe_block_forward/backward with ckpt (blocks.cpp:339-377; test_model.cpp:680-720):
    the replayed backward gives bitwise the same output, aux loss and gradients, and the
    layer holds fewer bytes between forward and backward."""
    b2, ctx = b2ctx
    dt = torch.bfloat16 if dtype == "bf16" else torch.float32
    cfg = b2.MoeConfig(n_experts=8, top_k=2, hidden=256, intermediate=128)
    S = 200
    gen = torch.Generator(device="cuda").manual_seed(33)
    mk = lambda shape, std: (torch.randn(shape, device="cuda", generator=gen) * std).to(dt)
    x, dout = mk((S, 256), 0.5), mk((S, 256), 0.3)
    router, gate, up, down = mk((256, 8), 0.1), mk((8, 256, 128), 0.1), mk((8, 256, 128), 0.1), mk((8, 128, 256), 0.1)
    res, held = [], []
    for ckpt in (False, True):
        layer = b2.MoeLayer(ctx, cfg, dt, S, checkpoint=ckpt)
        out = layer.forward(x, router, gate, up, down)
        aux = layer.aux_loss()
        held.append(layer.held_bytes())
        g = layer.backward(router, gate, up, down, dout, layer.aux_probs_grad(0.01))
        torch.cuda.synchronize()
        res.append(([out] + [g[k] for k in ("input", "router", "gate", "up", "down")], aux))
    (a, aux_a), (b, aux_b) = res
    for u, v in zip(a, b):
        assert torch.equal(u, v)
    assert aux_a == aux_b
    assert held[1] < held[0]


def test_shared_workspace_layers_match_private(b2ctx):
    """Two checkpointed layers on ONE activation workspace (forward 1, forward 2, backward 2,
    backward 1 — the order a model runs them) give the results of two private layers."""
    b2, ctx = b2ctx
    cfg = b2.MoeConfig(n_experts=16, top_k=4, hidden=256, intermediate=128)
    S = 300
    gen = torch.Generator(device="cuda").manual_seed(34)
    mk = lambda shape, std: (torch.randn(shape, device="cuda", generator=gen) * std).bfloat16()
    ws = [dict(router=mk((256, 16), 0.05), gate=mk((16, 256, 128), 0.05), up=mk((16, 256, 128), 0.05),
               down=mk((16, 128, 256), 0.05)) for _ in range(2)]
    x1, d2 = mk((S, 256), 1.0), mk((S, 256), 1.0)

    def run(l1, l2):
        w1, w2 = ws
        y1 = l1.forward(x1, w1["router"], w1["gate"], w1["up"], w1["down"])
        y2 = l2.forward(y1, w2["router"], w2["gate"], w2["up"], w2["down"])
        g2 = l2.backward(w2["router"], w2["gate"], w2["up"], w2["down"], d2)
        g1 = l1.backward(w1["router"], w1["gate"], w1["up"], w1["down"], g2["input"])
        torch.cuda.synchronize()
        return [y1, y2] + [g[k] for g in (g1, g2) for k in ("input", "router", "gate", "up", "down")]

    want = run(b2.MoeLayer(ctx, cfg, torch.bfloat16, S), b2.MoeLayer(ctx, cfg, torch.bfloat16, S))
    a = b2.MoeLayer(ctx, cfg, torch.bfloat16, S, checkpoint=True)
    b = b2.MoeLayer(ctx, cfg, torch.bfloat16, S, share_workspace=a, checkpoint=True)
    got = run(a, b)
    for u, v in zip(got, want):
        assert torch.equal(u, v)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("S,N,K", [(0, 8, 2), (1, 8, 2), (3, 1, 1), (65, 4, 4)])
def test_layer_edge_shapes(b2ctx, orc, dtype, S, N, K):
    """Empty and ragged inputs (S = 0, 1, odd), a single expert, top-k = all experts: the
    layer runs, matches the oracle, and an empty batch yields empty outputs and zero
    weight gradients."""
    b2, ctx = b2ctx
    dt = torch.bfloat16 if dtype == "bf16" else torch.float32
    H, I = 128, 64
    ocfg, bcfg = cfg_pair(n_experts=N, top_k=K, hidden=H, intermediate=I)
    rb = (lambda a: torch.from_numpy(np.ascontiguousarray(a)).bfloat16().float().numpy()) if dtype == "bf16" \
        else (lambda a: a)
    router, gate, up, down = (rb(t) for t in orc.expert_weights(ocfg, 1234, 0.05))
    x = rb(orc.normal((S, H), 77, 0, 1.0)) if S else np.zeros((0, H), np.float32)
    dout = rb(orc.normal((S, H), 78, 0, 1.0)) if S else np.zeros((0, H), np.float32)
    got = run_layer(b2, ctx, bcfg, dt, x, router, gate, up, down, dout, aux_coeff=0.0)
    if S == 0:
        assert got["out"].shape == (0, H) and got["input"].shape == (0, H)
        for k in ("gate", "up", "down", "router"):
            assert not np.any(got[k])
        return
    ref = orc.moe_layer(ocfg, S, x, router, gate, up, down, dout, aux_coeff=0.0)
    assert np.array_equal(got["indices"], ref["indices"])
    tol = 1e-4 if dtype == "f32" else 2e-2
    assert rel_err(got["out"], ref["out"]) <= tol
    assert rel_err(got["input"], ref["dx"]) <= tol
    for key, gkey in [("dgate", "gate"), ("dup", "up"), ("ddown", "down")]:
        assert (rel_err if dtype == "f32" else scale_err)(got[gkey], ref[key]) <= tol, key
