"""CPU pinning of the record-file restatement (oracle/moe_oracle.c: orc_record_file_bytes /
orc_record_file_parse) against the reference's RecordFileWriter / read_record_file
(reliability.cpp:222-320): byte-identical files for the reference's own RecordFiles tests
(test_reliability.cpp:205-278) and format edge cases, the same rejection message for every
corruption class, and the committed golden files written by the reference itself."""
import os
import zlib

import numpy as np
import pytest

import record_cases

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden")


@pytest.mark.parametrize("case", ["roundtrip", "rounding", "empty", "corrupt_base", "mixed"])
def test_oracle_reproduces_reference_golden_bytes(orc, tmp_path, case):
    recs = record_cases.cases(orc)[case]
    path = str(tmp_path / "o.bin")
    nbytes, crc = orc.record_file_write(path, recs)
    got = open(path, "rb").read()
    gold = open(os.path.join(GOLD, f"records_{case}.bin"), "rb").read()
    assert got == gold
    assert nbytes == len(gold) and crc == zlib.crc32(gold[:-4])
    if case == "empty":
        assert nbytes == 16  # header and footer only (test_reliability.cpp:242-249)


@pytest.mark.parametrize("case", ["roundtrip", "rounding", "mixed"])
def test_oracle_parse_matches_golden(orc, case):
    recs = record_cases.cases(orc)[case]
    cnt, vals = orc.record_file_read(os.path.join(GOLD, f"records_{case}.bin"))
    assert cnt == len(recs)
    want = []
    for _, dt, _, a in recs:
        a = np.asarray(a, np.float32)
        want.append(a if dt == 0 else np.array([orc._f("bf16_round")(float(x)) for x in a], np.float32))
    want = np.concatenate(want) if want else np.zeros(0, np.float32)
    assert np.array_equal(vals.view(np.uint32), want.view(np.uint32))


def test_oracle_matches_reference(orc, ref, tmp_path):
    for case, recs in record_cases.cases(orc).items():
        a, b = str(tmp_path / "o.bin"), str(tmp_path / "r.bin")
        assert orc.record_file_write(a, recs) == ref.record_file_write(b, recs), case
        assert open(a, "rb").read() == open(b, "rb").read(), case
        ca, va = orc.record_file_read(b)
        cb, vb = ref.record_file_read(a)
        assert ca == cb and np.array_equal(va.view(np.uint32), vb.view(np.uint32)), case


def test_corruptions_rejected_like_the_reference(orc, tmp_path):
    good = open(os.path.join(GOLD, "records_corrupt_base.bin"), "rb").read()
    path = str(tmp_path / "c.bin")
    for what, data in record_cases.corruptions(good):
        with open(path, "wb") as f:
            f.write(data)
        with pytest.raises(RuntimeError) as e:
            orc.record_file_read(path)
        assert str(e.value).endswith(WANT[what]), (what, str(e.value))


def test_corruption_messages_pinned_to_reference(ref, tmp_path):
    good = open(os.path.join(GOLD, "records_corrupt_base.bin"), "rb").read()
    path = str(tmp_path / "c.bin")
    for what, data in record_cases.corruptions(good):
        with open(path, "wb") as f:
            f.write(data)
        with pytest.raises(RuntimeError) as e:
            ref.record_file_read(path)
        assert str(e.value).endswith(path + ": " + WANT[what]), (what, str(e.value))


# read_record_file's message per corruption class (reliability.cpp:274-319)
WANT = {"flipped payload bit": "checksum mismatch", "truncated": "checksum mismatch",
        "short header": "truncated header", "wrong magic": "bad magic", "wrong version": "unsupported version",
        "count past the end": "truncated record", "trailing bytes": "trailing bytes after last record",
        "oversized name": "oversized record name", "unknown dtype": "unknown dtype",
        "too many dims": "too many dimensions"}
