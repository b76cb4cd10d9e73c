"""The CUDA path (through the C-ABI) on the committed golden vectors of the UNMODIFIED
reference (tests/golden/, see make_golden.py). fp32 mode: routing bit-exact, every output
and gradient within 1e-4 rel_err (tests/test_util.hpp:15-18 metric). EP = 1 fixtures; the
EP = 2 fixture runs in tests/test_gpu_ep.py's multi-process harness."""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from test_golden import ART_KEYS, LAYER_FILES, layer_inputs, load  # noqa: E402

pytestmark = pytest.mark.gpu
TOL = 1e-4


def rel_err(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b) / np.maximum(1.0, np.maximum(np.abs(a), np.abs(b))))) if a.size else 0.0


@pytest.mark.parametrize("path", [p for p in LAYER_FILES if "ep2" not in p], ids=lambda p: os.path.basename(p)[:-4])
def test_cuda_layer_matches_reference_golden(orc, path):
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2604_00785_b200 as b2
    g = load(path)
    cfg, s, x, router, gate, up, down, dout = layer_inputs(orc, g)
    bcfg = b2.MoeConfig(n_experts=cfg.n_experts, top_k=cfg.top_k, hidden=cfg.hidden, intermediate=cfg.intermediate,
                        ep=1, token_block=cfg.token_block, normalize_topk=bool(cfg.normalize_topk))
    ctx = b2.Context(0)
    tt = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    X, R, G, U, D, DO = map(tt, (x, router, gate, up, down, dout))
    layer = b2.MoeLayer(ctx, bcfg, torch.float32, s)
    out = layer.forward(X, R, G, U, D, fur=bool(g["fur"]))
    apg = layer.aux_probs_grad(float(g["aux_coeff"])) if float(g["aux_coeff"]) else None
    grads = layer.backward(R, G, U, D, DO, apg)
    torch.cuda.synchronize()
    probs, w, idx = layer.routing()
    assert np.array_equal(idx, g["indices"])
    assert np.array_equal(w, g["weights"])
    assert np.array_equal(probs, g["probs"])
    arts = layer.artifacts()
    for k in ART_KEYS:
        assert np.array_equal(np.asarray(arts[k]), g[f"art0_{k}"]), k
    assert rel_err(layer.aux_loss(), g["aux"][0]) <= TOL
    for key, got in (("out", out), ("dx", grads["input"]), ("drouter", grads["router"]), ("dgate", grads["gate"]),
                     ("dup", grads["up"]), ("ddown", grads["down"])):
        want = g[key][0] if key == "drouter" else g[key]
        e = rel_err(got.cpu().numpy(), want)
        assert e <= TOL, f"{key}: rel_err {e}"
