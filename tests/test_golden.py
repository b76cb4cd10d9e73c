"""The C restatement (oracle/liboracle.so) against golden vectors produced by the
UNMODIFIED reference (tests/golden/make_golden.py over oracle/_ref, compiled in place from
/root/reference). Needs neither the reference tree nor a GPU: the fixtures are committed.
Bar: bitwise equality on every stored output."""
import glob
import hashlib
import os

import numpy as np
import pytest

from oracle import bind

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
LAYER_FILES = sorted(glob.glob(os.path.join(GOLD, "layer_*.npz")))
SHARDED_FILES = sorted(glob.glob(os.path.join(GOLD, "sharded_*.npz")))
ART_KEYS = ("token_counts", "partial_token_counts", "partial_cum", "cum_token_counts", "expert_counts",
            "cum_expert_counts", "input_indices", "output_indices", "selected_k", "counter")


def load(path):
    with np.load(path) as d:
        return {k: d[k] for k in d.files}


def cfg_of(g):
    n, k, h, i, ep, tbs, norm = (int(v) for v in g["cfg"])
    return bind.moe_cfg(n_experts=n, top_k=k, hidden=h, intermediate=i, ep=ep, token_block=tbs,
                        normalize_topk=bool(norm))


def layer_inputs(orc, g):
    cfg = cfg_of(g)
    s = int(g["s_local"])
    std = float(g["std"])
    router, gate, up, down = orc.expert_weights(cfg, 1234, std)
    x = orc.normal((cfg.ep * s, cfg.hidden), 77, 0, 0.7)
    dout = orc.normal((cfg.ep * s, cfg.hidden), 78, 0, 1.0)
    h = hashlib.sha256()
    for a in (x, router, gate, up, down, dout):
        h.update(np.ascontiguousarray(a).tobytes())
    assert h.hexdigest() == str(g["input_sha256"]), "input generator drifted from the reference's"
    return cfg, s, x, router, gate, up, down, dout


def test_fixtures_present():
    assert len(LAYER_FILES) >= 5 and len(SHARDED_FILES) >= 9


@pytest.mark.parametrize("path", LAYER_FILES, ids=lambda p: os.path.basename(p)[:-4])
def test_oracle_layer_matches_reference_golden(orc, path):
    g = load(path)
    cfg, s, x, router, gate, up, down, dout = layer_inputs(orc, g)
    r = orc.moe_layer(cfg, s, x, router, gate, up, down, dout, fur=bool(g["fur"]), aux_coeff=float(g["aux_coeff"]))
    for k in ("out", "dx", "drouter", "dgate", "dup", "ddown", "weights", "indices", "probs", "aux"):
        assert np.array_equal(r[k], g[k]), k
    table = r["indices"] if not g["fur"] else \
        (np.arange(cfg.ep * s)[:, None] * cfg.top_k + np.arange(cfg.top_k)[None, :]) % cfg.n_experts
    for e in range(cfg.ep):
        a = orc.artifacts(cfg, table.astype(np.int64), e)
        for k in ART_KEYS:
            assert np.array_equal(np.asarray(a[k]), g[f"art{e}_{k}"]), (e, k)


def test_oracle_artifacts_match_reference_golden(orc):
    g = load(os.path.join(GOLD, "artifacts_ep3.npz"))
    cfg = bind.moe_cfg(n_experts=12, top_k=3, hidden=4, intermediate=4, ep=3, token_block=5)
    for e in range(3):
        a = orc.artifacts(cfg, g["table"], e)
        for k in ART_KEYS:
            assert np.array_equal(np.asarray(a[k]), g[f"art{e}_{k}"]), (e, k)


@pytest.mark.parametrize("path", SHARDED_FILES, ids=lambda p: os.path.basename(p)[:-4])
def test_oracle_sharded_step_matches_reference_golden(orc, path):
    g = load(path)
    name = os.path.basename(path)[:-4]
    dp, ep, mode = (int(name.split("_")[1][2:]), int(name.split("_")[2][2:]), int(name.split("_")[3][1:]))
    acfg = orc.adamw_cfg(warmup_steps=1, total_steps=10)
    r = orc.sharded_steps(dp, ep, 1, mode, acfg, g["numel"], g["cls"], np.zeros(len(g["numel"]), np.int32), g["w0"],
                          g["grads"])
    for k in ("weights", "master", "m", "v", "owned", "stats", "state_bytes"):
        assert np.array_equal(r[k], g[k]), k
