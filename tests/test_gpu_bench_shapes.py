"""Parity at the shapes bench.py measures (VERDICT r1 "What's missing" 1).

Config B (BASELINE.json configs[1]): the OLMoE-1B-7B layer, H=2048, N=64, K=8, I=1024.
Config E (configs[4]): the Mula-20B-A2B layer, H=2048, N=96, K=8, I=1024, Zipf-skewed routing.
Both run the full fast_moe_forward + fast_moe_backward (moe.hpp:344-466) through the C-ABI
and are compared with the CPU oracle on identical inputs (the reference's generators,
init_expert_weights moe.hpp:500-523 and normal_init, rounded to bf16 for the bf16 path):

  * routing indices, weights and every RoutingArtifacts array: bit-exact;
  * bf16 path vs the fp32 oracle: out / dX within 2e-2 rel_err elementwise
    (tests/test_util.hpp:15-18 metric), weight and router grads within 2e-2 of the
    tensor scale (long bf16 reductions);
  * fp32 path (SIMT mode): every output and gradient within 1e-4 rel_err;
  * the forward output also against the dense per-token oracle reference_moe_forward
    (moe.hpp:471-497; the reference's own check is test_moe.cpp:451-490 at 1e-5 in fp32).

At these sizes the GEMMs run long K loops (32 k-blocks at H=2048), many tiles per
persistent CTA and the TMA ring wraps over many tiles — the regime the small cases skip.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import bind

pytestmark = pytest.mark.gpu

TOL_F32 = 1e-4
TOL_BF16 = 2e-2
H, I, K = 2048, 1024, 8


def rel_err(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b) / np.maximum(1.0, np.maximum(np.abs(a), np.abs(b))))) if a.size else 0.0


def scale_err(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-30)) if a.size else 0.0


def bf16_round(a):
    return torch.from_numpy(np.ascontiguousarray(a)).bfloat16().float().numpy()


@pytest.fixture(scope="module")
def b2ctx():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2604_00785_b200 as b2
    return b2, b2.Context(0)


_WEIGHTS = {}


def weights(orc, n, bf16):
    """init_expert_weights (moe.hpp:500-523), seed 1234, sigma 0.02, full expert set."""
    key = (n, bf16)
    if key not in _WEIGHTS:
        cfg = bind.moe_cfg(n_experts=n, top_k=K, hidden=H, intermediate=I)
        w = orc.expert_weights(cfg, 1234, 0.02)
        _WEIGHTS.clear()  # one config resident at a time (config E fp32 weights are 2.4 GB)
        _WEIGHTS[key] = tuple(bf16_round(t) for t in w) if bf16 else w
    return _WEIGHTS[key]


def run_layer(b2, ctx, n, dtype, x, router, gate, up, down, dout, aux_coeff=0.01):
    cfg = b2.MoeConfig(n_experts=n, top_k=K, hidden=H, intermediate=I)
    tt = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda().to(dtype)
    X, R, G, U, D, DO = map(tt, (x, router, gate, up, down, dout))
    layer = b2.MoeLayer(ctx, cfg, dtype, x.shape[0])
    out = layer.forward(X, R, G, U, D)
    apg = layer.aux_probs_grad(aux_coeff)
    grads = layer.backward(R, G, U, D, DO, apg)
    torch.cuda.synchronize()
    res = {k: v.float().cpu().numpy() for k, v in grads.items()}
    res["out"] = out.float().cpu().numpy()
    res["probs"], res["weights"], res["indices"] = layer.routing()
    res["artifacts"] = layer.artifacts()
    res["aux"] = layer.aux_loss()
    layer.close()
    return res


def compare_artifacts(got, want):
    for key in ("token_counts", "partial_token_counts", "partial_cum", "cum_token_counts", "expert_counts",
                "cum_expert_counts", "input_indices", "output_indices", "selected_k", "counter"):
        assert np.array_equal(np.asarray(got[key]), np.asarray(want[key])), key
    assert got["rt"] == want["rt"] and got["th"] == want["th"]


def check_layer(orc, n, got, ref, x, gate, up, down, tol, grad_metric):
    ocfg = bind.moe_cfg(n_experts=n, top_k=K, hidden=H, intermediate=I)
    assert np.array_equal(got["indices"], ref["indices"])
    assert np.array_equal(got["weights"], ref["weights"])
    compare_artifacts(got["artifacts"], orc.artifacts(ocfg, ref["indices"], 0))
    assert rel_err(got["aux"], ref["aux"][0]) <= 1e-6
    errs = {"out": rel_err(got["out"], ref["out"]), "dx": rel_err(got["input"], ref["dx"])}
    for key, gkey in [("drouter", "router"), ("dgate", "gate"), ("dup", "up"), ("ddown", "down")]:
        want = ref[key][0] if key == "drouter" else ref[key]
        errs[key] = grad_metric(got[gkey], want)
    # the dense per-token oracle (moe.hpp:471-497) on the same routing: an independent
    # restatement of the forward (k-order accumulation instead of the expert-sorted one)
    dense = orc.dense_moe_forward(ocfg, x, gate, up, down, ref["weights"], ref["indices"])
    errs["out_vs_dense"] = rel_err(got["out"], dense)
    bad = {k: v for k, v in errs.items() if v > tol}
    assert not bad, f"over {tol}: {bad} (all: {errs})"
    return errs


@pytest.mark.parametrize("S", [512])
def test_config_b_bf16_layer(b2ctx, orc, S):
    """Config B dims, bf16 tensor-core path, vs the fp32 oracle on the same bf16 inputs."""
    b2, ctx = b2ctx
    N = 64
    ocfg = bind.moe_cfg(n_experts=N, top_k=K, hidden=H, intermediate=I)
    router, gate, up, down = weights(orc, N, True)
    x = bf16_round(orc.normal((S, H), 77, 0, 1.0))
    dout = bf16_round(orc.normal((S, H), 78, 0, 1.0))
    ref = orc.moe_layer(ocfg, S, x, router, gate, up, down, dout, aux_coeff=0.01)
    got = run_layer(b2, ctx, N, torch.bfloat16, x, router, gate, up, down, dout)
    errs = check_layer(orc, N, got, ref, x, gate, up, down, TOL_BF16, scale_err)
    print("config B bf16", errs)


def test_config_b_fp32_layer(b2ctx, orc):
    """Config B dims in the fp32 (SIMT) mode: every output and gradient within 1e-4."""
    b2, ctx = b2ctx
    N, S = 64, 256
    ocfg = bind.moe_cfg(n_experts=N, top_k=K, hidden=H, intermediate=I)
    router, gate, up, down = weights(orc, N, False)
    x = orc.normal((S, H), 77, 0, 1.0)
    dout = orc.normal((S, H), 78, 0, 1.0)
    ref = orc.moe_layer(ocfg, S, x, router, gate, up, down, dout, aux_coeff=0.01)
    got = run_layer(b2, ctx, N, torch.float32, x, router, gate, up, down, dout)
    errs = check_layer(orc, N, got, ref, x, gate, up, down, TOL_F32, rel_err)
    print("config B fp32", errs)


def zipf_inputs(S, N, s, seed=4242):
    """Config E routing (logits[t,e] = log z_e + noise, z_e ∝ (e+1)^-s, identity
    expert permutation so the hottest experts sit first) through a router of realistic
    magnitude: tokens x ~ N(1, 1) (mean-shifted), Wr = column-centred N(0, σ) + log z_e / H with
    σ = 1.2825 / sqrt(H) (the Gumbel noise's std). Then x·Wr = mean(x_t) · log z_e + N(0, 1.28²):
    Gumbel-top-k-like skew (s = 1.2: max/mean rows per expert 11.9 at 16k tokens) with O(0.03)
    router weights. (Embedding the logits in x with an identity router instead puts O(1)
    weights on the router, where the bf16 path's top-k-weight gradient — a dot with the bf16
    mlp_out — is amplified into dX: the bf16 floor, tools/parity_floor.py.)"""
    rng = np.random.default_rng(seed)
    z = (np.arange(N) + 1.0) ** -s
    z /= z.sum()
    x = (rng.standard_normal((S, H)) + 1.0).astype(np.float32)
    wn = rng.standard_normal((H, N)) * (1.2825 / np.sqrt(H))
    wn -= wn.mean(0, keepdims=True)
    router = (wn + np.log(z)[None, :] / H).astype(np.float32)
    return x, router


@pytest.mark.parametrize("s", [0.0, 1.2])
def test_config_e_bf16_zipf_layer(b2ctx, orc, s):
    """Config E dims (N=96) under uniform (s=0) and skewed (s=1.2) routing."""
    b2, ctx = b2ctx
    N, S = 96, 512
    ocfg = bind.moe_cfg(n_experts=N, top_k=K, hidden=H, intermediate=I)
    _, gate, up, down = weights(orc, N, True)
    x, router = zipf_inputs(S, N, s)
    x, router = bf16_round(x), bf16_round(router)
    dout = bf16_round(orc.normal((S, H), 78, 0, 1.0))
    ref = orc.moe_layer(ocfg, S, x, router, gate, up, down, dout, aux_coeff=0.01)
    counts = np.bincount(ref["indices"].ravel(), minlength=N)
    if s > 0:
        assert counts.max() >= 5 * counts.mean(), counts
    got = run_layer(b2, ctx, N, torch.bfloat16, x, router, gate, up, down, dout)
    errs = check_layer(orc, N, got, ref, x, gate, up, down, TOL_BF16, scale_err)
    for e in np.where(counts == 0)[0]:  # empty experts: exactly zero weight gradients
        assert not got["gate"][e].any() and not got["up"][e].any() and not got["down"][e].any()
    print(f"config E bf16 s={s}", errs)


@pytest.mark.parametrize("T,N,Kk,tbs", [(40000, 64, 8, 8), (70001, 96, 8, 3), (131072, 64, 8, 8)])
def test_routing_artifacts_large_tables_bit_exact(b2ctx, orc, T, N, Kk, tbs):
    """Tables past one block-scan round (16,384 tokens) and past one 256-chunk per-expert
    pass: the cross-round carry of cum_expert_counts and the second per-expert pass
    (index.cu), bitwise against count_tokens + generate_indices (moe.hpp:122-197). The
    last case is config B's full gathered table."""
    b2, ctx = b2ctx
    rng = np.random.default_rng(T)
    idx = np.argsort(rng.random((T, N)), axis=1)[:, :Kk].astype(np.int64)
    idx[: T // 3] = np.minimum(idx[: T // 3], 5)  # hot experts + repeated ids per token
    cfg_kw = dict(n_experts=N, top_k=Kk, hidden=8, intermediate=8, token_block=tbs)
    ocfg, bcfg = bind.moe_cfg(**cfg_kw), b2.MoeConfig(**cfg_kw)
    t = torch.from_numpy(idx.astype(np.int32)).cuda()
    compare_artifacts(b2.routing_artifacts(ctx, bcfg, t, 0), orc.artifacts(ocfg, idx, 0))
