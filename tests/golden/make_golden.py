"""Generates tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref/libref_optimus.so,
compiled in place from /root/reference/proj/src by oracle/Makefile). Run in the build
container, where /root/reference exists:

    make -C oracle && python tests/golden/make_golden.py

Inputs are regenerated from seeds by the reference's own generators (normal_init,
init_expert_weights: common.hpp:83-87, moe.hpp:500-523); each fixture stores the seeds,
a sha256 of the generated input bytes (so a drifting generator is caught) and the
reference's outputs. tests/test_golden.py checks the C restatement (oracle/liboracle.so)
bitwise against them on CPU; tests/test_gpu_golden.py checks the CUDA path."""
import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import bind  # noqa: E402

# small MoE layer cases (fp32 reference): name -> (cfg kwargs, s_local, fur, aux_coeff, weight std)
LAYERS = {
    "layer_a_small": (dict(n_experts=8, top_k=2, hidden=32, intermediate=48, ep=1, token_block=8), 64, False, 0.01, 0.2),
    "layer_ep2": (dict(n_experts=8, top_k=2, hidden=32, intermediate=24, ep=2, token_block=4), 24, False, 0.01, 0.2),
    "layer_norm_topk": (dict(n_experts=6, top_k=3, hidden=20, intermediate=12, ep=1, token_block=3,
                             normalize_topk=True), 37, False, 0.0, 0.2),
    "layer_fur": (dict(n_experts=8, top_k=2, hidden=16, intermediate=24, ep=1, token_block=4), 16, True, 0.0, 0.2),
    "layer_olmoe_dims_tiny": (dict(n_experts=64, top_k=8, hidden=32, intermediate=16, ep=1, token_block=8), 32,
                              False, 0.01, 0.05),
}


def digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def layer_inputs(o, cfg, s_local, std):
    T = cfg.ep * s_local
    router, gate, up, down = o.expert_weights(cfg, 1234, std)
    x = o.normal((T, cfg.hidden), 77, 0, 0.7)
    dout = o.normal((T, cfg.hidden), 78, 0, 1.0)
    return x, router, gate, up, down, dout


def main():
    if not bind.have_ref():
        sys.exit("oracle/_ref/libref_optimus.so missing: run `make -C oracle` where /root/reference exists")
    ref = bind.get("ref")
    for name, (kw, s_local, fur, aux, std) in LAYERS.items():
        cfg = bind.moe_cfg(**kw)
        x, router, gate, up, down, dout = layer_inputs(ref, cfg, s_local, std)
        r = ref.moe_layer(cfg, s_local, x, router, gate, up, down, dout, fur=fur, aux_coeff=aux)
        table = r["indices"] if not fur else \
            (np.arange(cfg.ep * s_local)[:, None] * cfg.top_k + np.arange(cfg.top_k)[None, :]) % cfg.n_experts
        arts = [ref.artifacts(cfg, table.astype(np.int64), e) for e in range(cfg.ep)]
        out = dict(cfg=np.array([kw.get(k, 0) for k in ("n_experts", "top_k", "hidden", "intermediate", "ep",
                                                        "token_block")] + [int(kw.get("normalize_topk", False))]),
                   s_local=s_local, fur=int(fur), aux_coeff=aux, std=std,
                   input_sha256=digest(x, router, gate, up, down, dout), **r)
        for e, a in enumerate(arts):
            for k, v in a.items():
                out[f"art{e}_{k}"] = np.asarray(v)
        np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
        print(name, {k: np.asarray(v).shape for k, v in r.items()})

    # routing-artifact stress: repeated experts across tokens, many token blocks, ep ranks
    rng = np.random.default_rng(7)
    cfg = bind.moe_cfg(n_experts=12, top_k=3, hidden=4, intermediate=4, ep=3, token_block=5)
    table = np.stack([rng.choice(12, 3, replace=False) for _ in range(97)]).astype(np.int64)
    out = dict(table=table)
    for e in range(3):
        for k, v in ref.artifacts(cfg, table, e).items():
            out[f"art{e}_{k}"] = np.asarray(v)
    np.savez_compressed(os.path.join(HERE, "artifacts_ep3.npz"), **out)

    # sharded AdamW (ShardedOptimizer::step, optim.cpp:130-194) on two steps, every mode
    numel = np.array([10, 7, 33, 5], np.int64)
    cls = np.array([0, 1, 1, 0], np.int32)  # non-expert / expert (ReplicationClass)
    tps = np.array([0, 0, 0, 0], np.int32)
    for dp, ep in ((1, 1), (2, 2), (1, 4)):
        W = dp * ep
        total = int(numel.sum())
        w0 = np.stack([ref.normal((total,), 402, 1, 0.05)] * W)
        grads = np.stack([np.stack([ref.normal((total,), ref.hash_mix(s, r), 3, 1e-3) for r in range(W)])
                          for s in range(2)])
        for mode in (0, 1, 2):
            acfg = ref.adamw_cfg(warmup_steps=1, total_steps=10)
            r = ref.sharded_steps(dp, ep, 1, mode, acfg, numel, cls, tps, w0, grads)
            np.savez_compressed(os.path.join(HERE, f"sharded_dp{dp}_ep{ep}_m{mode}.npz"), numel=numel, cls=cls,
                                w0=w0, grads=grads, **r)

    # record files (RecordFileWriter, reliability.cpp:222-270): the reference's own test
    # cases plus format edge cases, written by the reference itself
    sys.path.insert(0, os.path.dirname(HERE))
    import record_cases
    for name, recs in record_cases.cases(ref).items():
        ref.record_file_write(os.path.join(HERE, f"records_{name}.bin"), recs)
    print("ok")


if __name__ == "__main__":
    main()
