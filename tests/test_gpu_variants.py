"""The opt-in kernel variants compute bit-identical results to the defaults.

Each A/B hook swaps a kernel for another schedule of the same arithmetic, so outputs must be
bitwise equal: B2_GEMM_MC=2 (A operand multicast across two CTA pairs), B2_LOGITS_IMPL=t42 (the
token-paired router-logits kernel), B2_ADAMW_IMPL=stream (the TMA-streamed AdamW). Each variant
runs tests/variant_worker.py in its own process (the hooks are read once per process).
"""
import os
import subprocess
import sys
import tempfile

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def run_variant(td, env_extra):
    out = os.path.join(td, "_".join(f"{k}{v}" for k, v in env_extra.items()) or "default") + ".npz"
    env = dict(os.environ, **env_extra)
    subprocess.run([sys.executable, os.path.join(HERE, "variant_worker.py"), out], env=env, check=True, timeout=600)
    return dict(np.load(out))


@pytest.fixture(scope="module")
def default_run():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    with tempfile.TemporaryDirectory() as td:
        yield run_variant(td, {})


@pytest.mark.parametrize("env", [{"B2_GEMM_MC": "2"}, {"B2_LOGITS_IMPL": "t42"}, {"B2_ADAMW_IMPL": "stream"}],
                         ids=lambda e: ",".join(f"{k}={v}" for k, v in e.items()))
def test_variant_bitwise(default_run, env):
    with tempfile.TemporaryDirectory() as td:
        got = run_variant(td, env)
    assert set(got) == set(default_run)
    for k in default_run:
        assert np.array_equal(got[k], default_run[k]), k
