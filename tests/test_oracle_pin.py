"""Pins the CPU oracle (oracle/moe_oracle.c) before anything trusts it.

1. Known-answer vectors transcribed from the reference's own tests
   (test_moe.cpp, test_tensor.cpp, test_optim.cpp under /root/reference/proj/tests).
2. Bitwise equality with the reference itself (oracle/_ref, compiled in place)
   on seeded random cases covering every hot-path entry point.
CPU only.
"""
import math

import numpy as np
import pytest

from oracle import bind


# ---------------------------------------------------------------- known answers

def four_token_cfg(tbs=8):
    # test_moe.cpp:18-27
    return bind.moe_cfg(n_experts=4, top_k=2, hidden=4, intermediate=4, ep=2, token_block=tbs)


FOUR = np.array([[0, 1], [0, 2], [1, 3], [2, 3]], np.int64)  # test_moe.cpp:14-16


@pytest.mark.parametrize("which", ["orc", "ref"])
def test_four_token_counts_and_indices(which):
    if which == "ref" and not bind.have_ref():
        pytest.skip("no reference build")
    o = bind.get(which)
    a = o.artifacts(four_token_cfg(), FOUR, 0)
    # test_moe.cpp:44-55
    assert a["token_counts"].tolist() == [2, 2]
    assert a["expert_counts"].tolist() == [2, 1, 1, 0]
    assert a["cum_token_counts"].tolist() == [0, 2, 4]
    assert a["cum_expert_counts"].tolist() == [0, 2, 3, 4, 4]
    assert a["rt"] == 4
    # test_moe.cpp:110-119
    assert a["input_indices"].tolist() == [0, 1, 0, 2]
    assert a["output_indices"].tolist() == [0, 2, 1, 3]
    assert a["selected_k"].tolist() == [0, 1, 0, 0]
    a1 = o.artifacts(four_token_cfg(), FOUR, 1)
    assert a1["token_counts"].tolist() == [2, 2] and a1["rt"] == 4
    # cursors end at partial boundaries (test_moe.cpp:121-128)
    a2 = o.artifacts(four_token_cfg(1), FOUR, 0)
    for ln in range(2):
        for tid in range(a2["th"]):
            assert a2["counter"][ln, tid] == a2["partial_cum"][ln * a2["th"] + tid + 1]
    # token-block invariance (test_moe.cpp:193-207)
    for tbs in (1, 2, 3, 4):
        b = o.artifacts(four_token_cfg(tbs), FOUR, 0)
        assert b["th"] == (4 + tbs - 1) // tbs
        for k in ("input_indices", "output_indices", "selected_k", "cum_token_counts"):
            assert b[k].tolist() == a[k].tolist()


def test_no_local_selection_and_out_of_range(orc):
    cfg = four_token_cfg()
    cfg.top_k = 1
    a = orc.artifacts(cfg, np.array([[2], [3], [2]], np.int64), 0)  # test_moe.cpp:57-66
    assert a["rt"] == 0 and a["token_counts"].tolist() == [0, 0]
    with pytest.raises(RuntimeError):  # test_moe.cpp:105-108
        orc.artifacts(four_token_cfg(), np.array([[0, 1], [2, 7]], np.int64), 0)


def test_topk_ties_and_softmax_extremes(orc):
    # test_tensor.cpp:207-215: ties go to the lower index
    _, vals, idx = orc.softmax_topk(np.log(np.array([[0.3, 0.3, 0.3, 0.1]], np.float32)), 2)
    assert idx.tolist() == [[0, 1]]
    # softmax [1000, 0] -> [1, 0] (test_tensor.cpp:155-165)
    p, _, _ = orc.softmax_topk(np.array([[1000.0, 0.0]], np.float32), 1)
    assert p.tolist() == [[1.0, 0.0]]


def test_bf16_round_to_nearest_even(orc):
    # test_tensor.cpp:337-347
    def rt(bits):
        f = np.array([bits], np.uint32).view(np.float32)[0]
        return int(np.array([orc._f("bf16_round")(float(f))], np.float32).view(np.uint32)[0]) >> 16

    assert rt(0x3F808000) == 0x3F80
    assert rt(0x3F818000) == 0x3F82
    assert rt(0x3F808001) == 0x3F81


def test_adamw_known_answers(orc):
    cfg = orc.adamw_cfg()
    # test_optim.cpp:83-98: g=1, lr=1e-3 -> -9.99e-4
    ms, _, _, _ = orc.adamw_update(np.zeros(1, np.float32), np.zeros(1, np.float32), np.zeros(1, np.float32),
                                   np.ones(1, np.float32), 1e-3, 0, cfg, False)
    assert abs(ms[0] - (-9.99e-4)) < 2e-6
    # decay alone (test_optim.cpp:100-111)
    st = [np.array([2.0], np.float32), np.zeros(1, np.float32), np.zeros(1, np.float32)]
    expect = np.float32(2.0)
    for s in range(3):
        st[0], st[1], st[2], _ = orc.adamw_update(st[0], st[1], st[2], np.zeros(1, np.float32), 1e-2, s, cfg, False)
        expect = np.float32(float(expect) - 1e-2 * 0.1 * float(expect))
    assert st[0][0] == expect
    # lr schedule (test_optim.cpp:14-28)
    assert orc.lr_at_step(0, cfg) == 0.0
    assert orc.lr_at_step(cfg.warmup_steps, cfg) == pytest.approx(4e-4, abs=0)
    assert orc.lr_at_step(cfg.total_steps + 12345, cfg) == 4e-5
    # shard_slice (test_optim.cpp:161-178)
    assert orc.shard_slice(10, 4, 0) == (0, 2)
    assert orc.shard_slice(10, 4, 2) == (4, 6)
    assert orc.shard_slice(10, 4, 3) == (6, 10)


def test_grad_norm_counts_each_logical_element_once(orc):
    # test_optim.cpp:361-385: dp=2, tp=2, SO, sqrt(51)
    W, numel = 4, [3, 4]
    w0 = np.zeros((W, 7), np.float32)
    g = np.zeros((1, W, 7), np.float32)
    for r in range(W):
        tp = r % 2
        w0[r, :3] = 1.0 if tp == 0 else 2.0
        g[0, r, :3] = 1.0 if tp == 0 else 2.0
        w0[r, 3:] = 0.5
        g[0, r, 3:] = 3.0
    cfg = orc.adamw_cfg(clip_after_warmup_only=0)
    res = orc.sharded_steps(2, 1, 2, 1, cfg, numel, [0, 0], [1, 0], w0, g)
    assert abs(res["stats"][0, 0, 1] - math.sqrt(51.0)) < 1e-12
    assert abs(res["stats"][0, 0, 2] - 1.0 / math.sqrt(51.0)) < 1e-12


def test_clip_schedule(orc):
    # test_optim.cpp:387-410
    cfg = orc.adamw_cfg(warmup_steps=2, total_steps=10)
    g = np.array([[[4.0]], [[4.0]], [[4.0]], [[0.5]]], np.float32)
    res = orc.sharded_steps(1, 1, 1, 0, cfg, [1], [0], [0], np.zeros((1, 1), np.float32), g)
    st = res["stats"][:, 0]
    assert st[0, 2] == 1.0 and st[0, 1] == 4.0
    assert st[2, 2] == 0.25
    assert st[3, 2] == 1.0 and st[3, 1] == 0.5


def _stable_sort_oracle(indices, n_start, nr):
    sels = [(int(e) - n_start, t, k) for t, row in enumerate(indices) for k, e in enumerate(row)
            if n_start <= e < n_start + nr]
    return sels, sorted(sels, key=lambda s: s[0])


def test_stable_sort_permutation_random(orc):
    # test_moe.cpp:130-191 with the reference's own RNG stream
    rng = np.random.default_rng(7)
    for _ in range(40):
        ep = int(rng.integers(1, 4))
        n = ep * int(rng.integers(1, 6))
        k = int(rng.integers(1, min(4, n) + 1))
        tbs = int(rng.integers(1, 7))
        T = int(rng.integers(1, 26))
        idx = np.stack([rng.permutation(n)[:k] for _ in range(T)]).astype(np.int64)
        rank = int(rng.integers(0, ep))
        cfg = bind.moe_cfg(n_experts=n, top_k=k, ep=ep, token_block=tbs)
        a = orc.artifacts(cfg, idx, rank)
        sels, by_e = _stable_sort_oracle(idx, rank * (n // ep), n // ep)
        assert a["rt"] == len(sels)
        assert a["input_indices"].tolist() == [s[1] for s in by_e]
        assert sorted(a["output_indices"].tolist()) == list(range(a["rt"]))
        for pos, s in enumerate(sels):
            assert a["selected_k"][pos] == s[2]
            row = a["output_indices"][pos]
            assert a["input_indices"][row] == s[1]
            assert a["cum_token_counts"][s[0]] <= row < a["cum_token_counts"][s[0] + 1]


# ---------------------------------------------------------------- bitwise vs the reference

@pytest.mark.parametrize("seed", range(6))
def test_routing_artifacts_bitwise_vs_reference(orc, ref, seed):
    rng = np.random.default_rng(100 + seed)
    ep = int(rng.integers(1, 5))
    n = ep * int(rng.integers(1, 5))
    k = int(rng.integers(1, n + 1))
    T = int(rng.integers(1, 60))
    # repeated experts per token allowed, like test_moe.cpp:84-103
    idx = rng.integers(0, n, size=(T, k)).astype(np.int64)
    cfg = bind.moe_cfg(n_experts=n, top_k=k, ep=ep, token_block=int(rng.integers(1, 9)))
    for r in range(ep):
        a, b = orc.artifacts(cfg, idx, r), ref.artifacts(cfg, idx, r)
        for key in a:
            assert np.array_equal(np.asarray(a[key]), np.asarray(b[key])), key


CASES = [
    dict(n_experts=8, top_k=2, hidden=32, intermediate=48, ep=1, token_block=8, s=21),
    dict(n_experts=8, top_k=2, hidden=32, intermediate=48, ep=2, token_block=3, s=13),
    dict(n_experts=12, top_k=3, hidden=24, intermediate=20, ep=4, token_block=5, s=9),
    dict(n_experts=6, top_k=2, hidden=16, intermediate=16, ep=1, token_block=2, s=17, normalize=True),
    dict(n_experts=8, top_k=2, hidden=16, intermediate=24, ep=2, token_block=4, s=8, fur=True),
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"ep{c['ep']}-n{c['n_experts']}")
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_moe_layer_bitwise_vs_reference(orc, ref, case, dtype):
    c = dict(case)
    s = c.pop("s")
    fur = c.pop("fur", False)
    norm = c.pop("normalize", False)
    cfg = bind.moe_cfg(normalize_topk=norm, **c)
    rw, g, u, d = orc.expert_weights(cfg, 1234, 0.2)
    x = orc.normal((cfg.ep * s, cfg.hidden), 77, 0, 0.7)
    dout = orc.normal((cfg.ep * s, cfg.hidden), 78, 0, 1.0)
    a = orc.moe_layer(cfg, s, x, rw, g, u, d, dout, fur=fur, aux_coeff=0.01, dtype=dtype)
    b = ref.moe_layer(cfg, s, x, rw, g, u, d, dout, fur=fur, aux_coeff=0.01, dtype=dtype)
    for key in a:
        assert np.array_equal(a[key], b[key]), key


@pytest.mark.parametrize("n,k,h,i,t", [(8, 2, 32, 48, 40), (64, 8, 64, 32, 97), (6, 6, 16, 8, 5)])
def test_dense_forward_bitwise_vs_reference_and_close_to_fast(orc, ref, n, k, h, i, t):
    """reference_moe_forward (moe.hpp:471-497): restatement == reference bitwise; fast path
    == dense within 1e-5 (the reference's own bar, test_moe.cpp:451-490)."""
    cfg = bind.moe_cfg(n_experts=n, top_k=k, hidden=h, intermediate=i)
    rw, g, u, d = orc.expert_weights(cfg, 1234, 0.2)
    x = orc.normal((t, h), 77, 0, 0.7)
    fast = orc.moe_layer(cfg, t, x, rw, g, u, d)
    a = orc.dense_moe_forward(cfg, x, g, u, d, fast["weights"], fast["indices"])
    b = ref.dense_moe_forward(cfg, x, g, u, d, fast["weights"], fast["indices"])
    assert np.array_equal(a, b)
    err = np.max(np.abs(a - fast["out"]) / np.maximum(1.0, np.maximum(np.abs(a), np.abs(fast["out"]))))
    assert err <= 1e-5


def test_dense_forward_rejects_bad_ids(orc):
    cfg = bind.moe_cfg(n_experts=4, top_k=2, hidden=4, intermediate=4)
    z = np.zeros((1, 4), np.float32)
    w = np.zeros((4, 4, 4), np.float32)
    with pytest.raises(RuntimeError, match="out of range"):
        orc.dense_moe_forward(cfg, z, w, w, w, np.ones((1, 2), np.float32), np.array([[0, 4]]))


@pytest.mark.parametrize("dp,ep,mode,bf16", [(1, 1, 1, True), (4, 1, 0, True), (4, 1, 1, True),
                                              (2, 2, 1, False), (2, 2, 2, False), (2, 2, 2, True),
                                              (1, 4, 2, True), (2, 1, 2, True)])
def test_sharded_steps_bitwise_vs_reference(orc, ref, dp, ep, mode, bf16):
    numel = [33, 30, 7]
    cls = [0, 1, 0]
    W, total = dp * ep, sum(numel)
    rng = np.random.default_rng(dp * 10 + ep + mode)
    w0 = np.zeros((W, total), np.float32)
    for r in range(W):
        e = r % ep
        w0[r, :33] = orc.normal((33,), 402, 1, 0.05)
        w0[r, 33:63] = orc.normal((30,), 403, 100 + e, 0.05)
        w0[r, 63:] = orc.normal((7,), 404, 2, 0.05)
    steps = 6
    g = rng.standard_normal((steps, W, total)).astype(np.float32)
    cfg = orc.adamw_cfg(warmup_steps=3, total_steps=100, peak_lr=1e-2, min_lr=1e-3, round_weights_bf16=int(bf16))
    a = orc.sharded_steps(dp, ep, 1, mode, cfg, numel, cls, [0, 0, 0], w0, g)
    b = ref.sharded_steps(dp, ep, 1, mode, cfg, numel, cls, [0, 0, 0], w0, g)
    for key in a:
        assert np.array_equal(a[key], b[key]), key


def test_so_equals_ddp_and_epso_close_to_so(orc):
    # test_optim.cpp:333-359
    numel, cls = [33, 30], [0, 1]

    def run(mode, dp, ep, bf16):
        W = dp * ep
        w0 = np.zeros((W, 63), np.float32)
        g = np.zeros((30, W, 63), np.float32)
        for r in range(W):
            e, d = r % ep, r // ep
            w0[r, :33] = orc.normal((33,), 402, 1, 0.05)
            w0[r, 33:] = orc.normal((30,), 403, 100 + e, 0.05)
            for s in range(30):
                salt = orc.hash_mix(s, d * 64 + e)
                g[s, r, :33] = orc.normal((33,), 400, salt)
                g[s, r, 33:] = orc.normal((30,), 401, salt)
        cfg = orc.adamw_cfg(warmup_steps=3, total_steps=100, peak_lr=1e-2, min_lr=1e-3, round_weights_bf16=int(bf16))
        return orc.sharded_steps(dp, ep, 1, mode, cfg, numel, cls, [0, 0], w0, g)

    ddp, so = run(0, 4, 1, True), run(1, 4, 1, True)
    assert np.array_equal(ddp["weights"], so["weights"])
    assert ddp["state_bytes"].sum() == 4 * 12 * 63 and so["state_bytes"].sum() == 12 * 63
    so2, epso = run(1, 2, 2, False), run(2, 2, 2, False)
    assert np.max(np.abs(so2["weights"] - epso["weights"]) / np.maximum(1, np.abs(so2["weights"]))) <= 1e-6
    assert so2["state_bytes"].sum() == 12 * (2 * 30 + 2 * 33)
    assert epso["state_bytes"].sum() == 12 * (2 * 30 + 33)
