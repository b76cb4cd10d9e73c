"""CPU checks of the drop-in boundary: libb2moe.so loads, exports every entry
point include/b2moe.h declares, the host-only helpers match the oracle, and compute
calls fail loudly (status 3) when no GPU is present — there is no CPU fallback."""
import ctypes as C
import os
import re

import pytest

import paper_2604_00785_b200 as b2

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared(header):
    src = open(os.path.join(ROOT, "include", header)).read()
    return sorted(set(re.findall(r"\b(b2x?_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = b2.lib()
    names = declared("b2moe.h") + declared("b2moe_testing.h")
    assert len(names) >= 30
    for n in names:
        assert hasattr(lib, n), n
    assert set(declared("b2moe.h")) == set(b2.SIGNATURES), "python bindings out of sync with the header"


def test_host_helpers_match_oracle(orc):
    cfg = b2.AdamWConfig()
    ocfg = orc.adamw_cfg()
    for s in (0, 1, 17, 2499, 2500, 2501, 50000, 100000, 123456):
        assert b2.lr_at_step(s, cfg) == orc.lr_at_step(s, ocfg)
    for numel in (1, 5, 16, 97, 10):
        for g in (1, 2, 3, 4, 8):
            for p in range(g):
                assert b2.shard_slice(numel, g, p) == orc.shard_slice(numel, g, p)
    with pytest.raises(b2.ContractError):
        b2.shard_slice(10, 4, 4)


def test_memory_report_matches_reference(orc):
    """memory_report (optim.cpp:196-221): the reference's known answer (7 B params under DDP need
    112 GB, test_optim.cpp:180-187), the C restatement and — when built — the reference itself,
    for every mode over DP x EP grids; the Mula-7B-A1B set fits one B200 (180 GB) under EPSO."""
    r = b2.memory_report(0, 7_000_000_000, 0, 1, 1)
    assert r["total_bytes"] == 112e9 and not r["feasible"]
    assert (r["weights_bytes"], r["master_bytes"], r["optim_bytes"]) == (14e9, 28e9, 56e9)
    z = b2.memory_report(0, 0, 2, 4, 2)
    assert z["total_bytes"] == 0 and z["feasible"]
    oracles = [orc]
    from oracle import bind
    if bind.have_ref():
        oracles.append(bind.get("ref"))
    for mode in (0, 1, 2):
        for dp, ep in ((1, 1), (2, 1), (1, 8), (2, 4), (4, 2), (8, 1), (3, 5)):
            got = b2.memory_report(6_442_450_944, 476_645_376, mode, dp, ep, 180.0)
            for o in oracles:
                assert got == o.memory_report(6_442_450_944, 476_645_376, mode, dp, ep, 180.0), (mode, dp, ep)
    assert b2.memory_report(6_442_450_944, 476_645_376, 2, 1, 1, 180.0)["feasible"]
    with pytest.raises(b2.ContractError):
        b2.memory_report(-1, 0, 2, 1, 1)


def test_lr_rejects_negative_step():
    assert b2.lr_at_step(-1, b2.AdamWConfig()) == -1.0
    assert "negative step" in b2.lib().b2_last_error().decode()


def test_compute_without_gpu_fails_loudly():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    lib = b2.lib()
    h = C.c_void_p()
    rc = lib.b2_ctx_create(0, None, 0, 1, 1, 1, 1, None, C.byref(h))
    assert rc == 3
    assert "no CUDA device" in lib.b2_last_error().decode()
    assert lib.b2_device_ok() == 0
