#!/usr/bin/env python
"""Where the bf16 layer's error sits relative to bf16's own floor (config B / config E dims).

Runs the bf16 layer on the GPU and the fp32 oracle on the same bf16 inputs (as
tests/test_gpu_bench_shapes.py does), then also an EMULATED bf16 forward in torch fp32 on
the GPU that rounds to bf16 exactly where the B200 path stores bf16 (G, U, H, Y, out) and
nowhere else. If the GPU's error matches the emulation's, it is the bf16 storage floor of
the algorithm, not a kernel defect. Prints the worst elements with their magnitudes.

  python tools/parity_floor.py --n 96 --zipf 0      # config E, uniform routing
  python tools/parity_floor.py --n 64               # config B
"""
import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle import bind  # noqa: E402
import paper_2604_00785_b200 as b2  # noqa: E402
from test_gpu_bench_shapes import H, I, K, bf16_round, rel_err, run_layer, zipf_inputs  # noqa: E402


def worst(name, got, want, n=5):
    d = np.abs(got.astype(np.float64) - want) / np.maximum(1.0, np.maximum(np.abs(got), np.abs(want)))
    flat = np.argsort(d.ravel())[::-1][:n]
    print(f"{name}: max rel_err {d.max():.3e}, 99.9% {np.quantile(d, 0.999):.3e}, median {np.median(d):.3e}")
    for f in flat:
        idx = np.unravel_index(f, d.shape)
        print(f"   at {idx}: got {got[idx]: .5f} want {want[idx]: .5f}")


def emulated_forward(x, gate, up, down, w, idx):
    """bf16 roundings at the B200 path's storage points, fp32 math in between."""
    dev = "cuda"
    X = torch.from_numpy(x).to(dev)
    out = torch.zeros_like(X)
    bf = lambda t: t.bfloat16().float()
    for e in np.unique(idx):
        rows, ks = np.nonzero(idx == e)
        xr = X[rows]
        g = bf(xr @ torch.from_numpy(gate[e]).to(dev))
        u = bf(xr @ torch.from_numpy(up[e]).to(dev))
        h = bf(torch.nn.functional.silu(g) * u)
        y = bf(h @ torch.from_numpy(down[e]).to(dev))
        out.index_put_((torch.from_numpy(rows).to(dev),), torch.from_numpy(w[rows, ks]).to(dev)[:, None] * y,
                       accumulate=True)
    return bf(out).cpu().numpy()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=96)
    ap.add_argument("--zipf", type=float, default=0.0)
    ap.add_argument("--s", type=int, default=512)
    ap.add_argument("--identity-router", action="store_true",
                    help="logits carried in x[:, :N] with Wr = [I; 0] (O(1) router weights)")
    a = ap.parse_args()
    orc = bind.get("orc")
    ctx = b2.Context(0)
    N, S = a.n, a.s
    ocfg = bind.moe_cfg(n_experts=N, top_k=K, hidden=H, intermediate=I)
    router, gate, up, down = (bf16_round(t) for t in orc.expert_weights(ocfg, 1234, 0.02))
    if a.identity_router:
        rng = np.random.default_rng(4242)
        z = (np.arange(N) + 1.0) ** -a.zipf
        z /= z.sum()
        x = rng.standard_normal((S, H)).astype(np.float32)
        x[:, :N] = np.log(z)[None, :] - np.log(-np.log(rng.uniform(1e-12, 1.0, (S, N))))
        router = np.zeros((H, N), np.float32)
        router[np.arange(N), np.arange(N)] = 1.0
        x, router = bf16_round(x), bf16_round(router)
    elif N == 96:
        x, router = zipf_inputs(S, N, a.zipf)
        x, router = bf16_round(x), bf16_round(router)
    else:
        x = bf16_round(orc.normal((S, H), 77, 0, 1.0))
    dout = bf16_round(orc.normal((S, H), 78, 0, 1.0))
    ref = orc.moe_layer(ocfg, S, x, router, gate, up, down, dout, aux_coeff=0.01)
    got = run_layer(b2, ctx, N, torch.bfloat16, x, router, gate, up, down, dout)
    print(f"N={N} zipf={a.zipf} S={S}: |x| max {np.abs(x).max():.2f}, |out| max {np.abs(ref['out']).max():.3f}, "
          f"|dx| max {np.abs(ref['dx']).max():.3f}")
    worst("out (GPU vs oracle)", got["out"], ref["out"])
    emu = emulated_forward(x, gate, up, down, ref["weights"], ref["indices"])
    worst("out (bf16 emulation vs oracle)", emu, ref["out"])
    worst("dx (GPU vs oracle)", got["input"], ref["dx"])
    print("drouter scale err", float(np.abs(got["router"] - ref["drouter"][0]).max() / np.abs(ref["drouter"][0]).max()))
    print("out rel_err vs oracle", rel_err(got["out"], ref["out"]))


if __name__ == "__main__":
    main()
