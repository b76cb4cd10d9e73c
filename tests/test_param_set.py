"""bench.py's EPSO parameter set against the reference's own Model::param_slots and count_params
(src/model.cpp:31-91, 189-229), through the reference compiled in place (oracle/_ref)."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


@pytest.mark.parametrize("ep", [1, 2, 4, 8])
def test_tiny_slots_match_reference(ref, ep):
    # mula-tiny (model.cpp:56-59): 2 layers, hidden 64, 4 x 16 heads, 8 experts of ffn 128, vocab 257
    for coord in range(ep):
        got = ref.param_slots("mula-tiny", ep, coord)
        assert got == bench.mula_param_set(2, 64, 4, 16, 128, 8, 257, ep), (ep, coord)


def test_7b_counts_match_reference(ref):
    total, _ = ref.count_params("mula-7b-a1b")
    slots = bench.mula7b_param_set()
    assert total == sum(n for n, _, _ in slots) == 6_919_096_320
    assert sum(n for n, e, _ in slots if e) == 6_442_450_944  # expert share
    for ep in (2, 4, 8):  # each EP rank: 1/ep of the experts, every non-expert parameter
        per = bench.mula7b_param_set(ep)
        assert sum(n for n, e, _ in per if e) * ep == 6_442_450_944
        assert sum(n for n, e, _ in per if not e) == 476_645_376
