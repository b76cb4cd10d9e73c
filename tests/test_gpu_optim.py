"""Single-GPU parity of the multi-tensor ShardedOptimizer step (optim.cpp:130-194) with the
oracle's ShardedOptimizer (oracle/moe_oracle.c, pinned bitwise to the reference), and the
soft-failure paths (reliability.cpp:706-723).

Bars: bf16 / fp32 grads, weights, fp32 masters and moments bitwise equal to the oracle
after several steps (warmup, clipping active); grad-norm statistics within 1e-12 relative
(the fp64 sum is reduced in a different, fixed order)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

# ragged sizes: a slice that is not a multiple of 4, one spanning several 64K chunks
NUMEL = [33, 130_001, 7, 4096, 70_000]
CLS = [0, 1, 0, 1, 1]


@pytest.fixture(scope="module")
def b2ctx():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2604_00785_b200 as b2
    return b2, b2.Context(0)


def make(orc, dtype, steps, seed=3):
    total = sum(NUMEL)
    w0 = np.concatenate([orc.normal((n,), 402 + p, 1, 0.05) for p, n in enumerate(NUMEL)])
    rng = np.random.default_rng(seed)
    grads = (rng.standard_normal((steps, total)) * 0.02).astype(np.float32)
    if dtype == torch.bfloat16:  # the oracle sees the same bf16-rounded values
        w0 = torch.from_numpy(w0).bfloat16().float().numpy()
        grads = torch.from_numpy(grads).bfloat16().float().numpy()
    return w0, grads


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32], ids=["bf16", "f32"])
@pytest.mark.parametrize("mode", [0, 1, 2], ids=["ddp", "so", "epso"])
def test_step_matches_oracle(b2ctx, orc, dtype, mode):
    b2, ctx = b2ctx
    steps = 5
    w0, grads = make(orc, dtype, steps)
    W = torch.from_numpy(w0).cuda().to(dtype)
    G = torch.zeros(W.numel(), dtype=dtype, device="cuda")
    params, off = [], 0
    for n, c in zip(NUMEL, CLS):
        params.append((W[off:off + n], G[off:off + n], c, 0))
        off += n
    cfg = b2.AdamWConfig(warmup_steps=2, total_steps=50, peak_lr=1e-2, min_lr=1e-3, clip_norm=1.0)
    opt = b2.ShardedOptimizer(ctx, cfg, params, mode)
    got = []
    for s in range(steps):
        G.copy_(torch.from_numpy(grads[s]).to(dtype))
        got.append(opt.step(stats=True))
    torch.cuda.synchronize()
    ocfg = orc.adamw_cfg(warmup_steps=2, total_steps=50, peak_lr=1e-2, min_lr=1e-3, clip_norm=1.0)
    ref = orc.sharded_steps(1, 1, 1, mode, ocfg, NUMEL, CLS, [0] * len(NUMEL), w0[None], grads[:, None, :])
    want_w = ref["weights"][0]
    if dtype == torch.bfloat16:
        assert np.array_equal(W.float().cpu().numpy(), want_w)
    else:
        assert np.array_equal(W.cpu().numpy(), want_w)
    ms = np.concatenate([opt.state(p)[0] for p in range(len(NUMEL))])
    m = np.concatenate([opt.state(p)[1] for p in range(len(NUMEL))])
    v = np.concatenate([opt.state(p)[2] for p in range(len(NUMEL))])
    assert np.array_equal(ms, ref["master"][0]) and np.array_equal(m, ref["m"][0]) and np.array_equal(v, ref["v"][0])
    for s, st in enumerate(got):
        lr, norm, clip = ref["stats"][s, 0]
        assert st["lr"] == lr and abs(st["grad_norm"] - norm) <= 1e-12 * norm and not st["nonfinite"]
        assert abs(st["clip_scale"] - clip) <= 1e-12
    assert any(st["clip_scale"] < 1.0 for st in got)  # clipping was exercised
    assert opt.state_bytes() == 12 * sum(NUMEL)
    assert opt.last_launches() > 0


def test_nonfinite_grad_is_detected_and_step_matches_reference(b2ctx, orc):
    """detect_soft_failure (reliability.cpp:706-723) flags a non-finite loss or grad; the step's
    fused scan reports it in the stats. Like the reference's ShardedOptimizer::step
    (optim.cpp:130-194) the step itself always applies the update and advances the step count
    (the training loop checks detect_soft_failure first, train.cpp:193-194), so a later step
    sees the same lr and bias corrections as the reference."""
    b2, ctx = b2ctx
    w0, grads = make(orc, torch.bfloat16, 2)
    W = torch.from_numpy(w0).cuda().bfloat16()
    G = torch.from_numpy(grads[0]).cuda().bfloat16()
    params, off = [], 0
    for n, c in zip(NUMEL, CLS):
        params.append((W[off:off + n], G[off:off + n], c, 0))
        off += n
    opt = b2.ShardedOptimizer(ctx, b2.AdamWConfig(warmup_steps=0), params, b2.EPSO)
    assert opt.detect_soft_failure(1.25, node=0) == -1
    assert opt.detect_soft_failure(float("nan"), node=0) == 0  # a non-finite loss is a failure too
    G[130_500] = float("inf")
    assert opt.detect_soft_failure(1.25, node=3) == 3
    st = opt.step(stats=True)
    torch.cuda.synchronize()
    assert st["nonfinite"] and st["step"] == 0
    st = opt.step(stats=True)
    assert st["step"] == 1  # the count advanced, as in the reference


def test_state_checkpoint_restore_continues_bitwise(b2ctx, orc):
    """gather_state / load_state (reliability.cpp:411-440, 658-667): a fresh optimizer
    restored from the assembled state (+ the step count) continues exactly like the
    original."""
    b2, ctx = b2ctx
    w0, grads = make(orc, torch.bfloat16, 6, seed=8)
    cfg = b2.AdamWConfig(warmup_steps=2, total_steps=50, peak_lr=1e-2, min_lr=1e-3)

    def build(w):
        W = torch.from_numpy(w).cuda().bfloat16()
        G = torch.zeros(W.numel(), dtype=torch.bfloat16, device="cuda")
        params, off = [], 0
        for n, c in zip(NUMEL, CLS):
            params.append((W[off:off + n], G[off:off + n], c, 0))
            off += n
        return W, G, b2.ShardedOptimizer(ctx, cfg, params, b2.EPSO)

    W, G, opt = build(w0)
    for s in range(3):
        G.copy_(torch.from_numpy(grads[s]).bfloat16())
        opt.step(stats=False)
    torch.cuda.synchronize()
    saved = [opt.gather_state(p, n) for p, n in enumerate(NUMEL)]
    W2, G2, opt2 = build(W.float().cpu().numpy())
    for p, st in enumerate(saved):
        opt2.load_state(p, *st)
    opt2.set_step_count(3)
    for s in range(3, 6):
        for G_, o in ((G, opt), (G2, opt2)):
            G_.copy_(torch.from_numpy(grads[s]).bfloat16())
            o.step(stats=False)
    torch.cuda.synchronize()
    assert torch.equal(W, W2)
    for p, n in enumerate(NUMEL):
        for a, b in zip(opt.gather_state(p, n), opt2.gather_state(p, n)):
            assert np.array_equal(a, b)


def _adversarial_state(n, seed):
    """master / exp_avg / exp_avg_sq / grad covering the update's corner cases: signed zeros,
    float subnormals, magnitudes from 1e-38 to 1e30, exact powers of two, v = 0 with m != 0,
    and a few non-finite values, mixed with ordinary training-scale values."""
    rng = np.random.default_rng(seed)

    def mixed(scale):
        x = (rng.standard_normal(n) * scale).astype(np.float32)
        pick = rng.integers(0, 12, n)
        x[pick == 0] = 0.0
        x[pick == 1] = -0.0
        x[pick == 2] = (rng.standard_normal((pick == 2).sum()) * 1e-40).astype(np.float32)  # subnormal
        x[pick == 3] = (10.0 ** rng.uniform(-38, 30, (pick == 3).sum()) * rng.choice([-1, 1], (pick == 3).sum()))
        x[pick == 4] = np.ldexp(1.0, rng.integers(-30, 10, (pick == 4).sum())).astype(np.float32)
        return x

    master = mixed(0.05)
    m = mixed(1e-3)
    v = np.abs(mixed(1e-6)).astype(np.float32)
    g = mixed(0.02)
    m[rng.integers(0, n, 8)] = 1e-3  # v stays 0 there when g is 0: the sqrt(0) branch
    for arr, val in ((g, np.inf), (g, np.nan), (master, -np.inf), (v, np.nan)):
        arr[rng.integers(0, n, 3)] = val
    return master, m, v, g


@pytest.mark.parametrize("wdt", ["f32", "bf16"])
@pytest.mark.parametrize("step,lr", [(0, 4e-4), (7, 1e-2), (2500, 0.0)])
def test_adamw_update_adversarial_bitwise(b2ctx, orc, wdt, step, lr):
    """adamw_update (optim.cpp:88-107) on corner-case states: the kernel's fast path (MUFU
    seeds + one Newton step, checked against the float rounding boundary) must fall back to
    the exactly rounded sequence wherever that check is not conclusive, so master, moments
    and weight are bit-identical to the reference's (NaN payloads aside)."""
    b2, ctx = b2ctx
    n = (1 << 20) + 4 if wdt == "bf16" else 200_003
    master, m, v, g = _adversarial_state(n, seed=step + 11)
    dt = torch.bfloat16 if wdt == "bf16" else torch.float32
    G = torch.from_numpy(g).to(dt).cuda()
    g_seen = G.float().cpu().numpy()
    dM, dm, dv = (torch.from_numpy(a.copy()).cuda() for a in (master, m, v))
    W = torch.empty(n, dtype=dt, device="cuda")
    cfg = b2.AdamWConfig()
    b2.adamw_update(ctx, dM, dm, dv, G, lr, step, cfg, W, round_bf16=True)
    torch.cuda.synchronize()
    rm, rmo, rv, rw = orc.adamw_update(master, m, v, g_seen, lr, step, orc.adamw_cfg(), round_bf16=True)
    for got, want in ((dM, rm), (dm, rmo), (dv, rv), (W.float(), rw)):
        got = got.cpu().numpy()
        nan = np.isnan(want)
        assert np.array_equal(np.isnan(got), nan)
        bad = got.view(np.uint32)[~nan] != want.view(np.uint32)[~nan]
        assert not bad.any(), f"{bad.sum()} of {n} differ"
