"""Record-file test cases shared by the CPU pinning tests, the golden generator and the
GPU tests. The first four are the reference's own RecordFiles tests
(/root/reference/proj/tests/test_reliability.cpp:205-278); ``mixed`` adds the edge
cases of the format (empty and 0-d records, NaN/Inf, ties, long names)."""
import zlib

import numpy as np

F32, BF16 = 0, 1


def _f(*v):
    return np.array(v, np.float32)


def cases(orc):
    """name -> [(record name, dtype, dims, f32 values)]; orc supplies bf16_round."""
    i12 = np.arange(12, dtype=np.float32)
    beta = np.array([orc._f("bf16_round")(float(np.float32(0.01) * v - np.float32(0.05))) for v in i12], np.float32)
    rng = np.random.default_rng(7)
    ties = np.array([1.00390625, 1.01171875, -1.00390625, 3.0e38, 1e-40, -0.0], np.float32)
    return {
        "roundtrip": [("alpha", F32, (2, 3), _f(1.5, -0.0, 3.25e-7, -42.0, 0.1, 2.0)),
                      ("beta", BF16, (3, 4), beta)],
        "rounding": [("x", BF16, (5,), _f(1.0000001, 3.14159265, -2.7182818, 1e-20, 65504.0))],
        "empty": [],
        "corrupt_base": [("x", F32, (20,), np.arange(20, dtype=np.float32) * np.float32(0.5))],
        "mixed": [("layer0.moe.gate.w16", BF16, (4, 8, 3), rng.standard_normal(96).astype(np.float32)),
                  ("layer0.moe.gate.master", F32, (96,), rng.standard_normal(96).astype(np.float32)),
                  ("nothing", F32, (0,), np.zeros(0, np.float32)),
                  ("zero_rows", BF16, (0, 5), np.zeros(0, np.float32)),
                  ("scalar", F32, (), _f(np.nan)),
                  ("specials", BF16, (8,), _f(np.nan, -np.nan, np.inf, -np.inf, 0.0, -0.0, 65504.0, 1e-45)),
                  ("ties", BF16, (6,), ties),
                  ("n" * 300, F32, (1, 1, 1, 1, 1, 1, 1, 2), _f(7.0, -7.0))],
    }


def _u32(v):
    return int(v).to_bytes(4, "little")


def _recrc(b: bytes) -> bytes:
    return b[:-4] + _u32(zlib.crc32(b[:-4]))


def corruptions(good: bytes):
    """(what, bytes) variants of one valid single-record file, each rejected by
    read_record_file (reliability.cpp:272-320) at a different check."""
    b = bytearray(good)
    flipped = bytearray(b)
    flipped[30] ^= 0x40
    out = [("flipped payload bit", bytes(flipped)), ("truncated", bytes(b[:-3])), ("short header", bytes(b[:15]))]
    wm = bytearray(b)
    wm[0] = ord("X")
    out.append(("wrong magic", bytes(wm)))
    wv = bytearray(b)
    wv[4:8] = _u32(2)
    out.append(("wrong version", _recrc(bytes(wv))))
    more = bytearray(b)
    more[8:12] = _u32(2)
    out.append(("count past the end", _recrc(bytes(more))))
    trail = bytes(b[:-4]) + b"\0\0\0\0" + bytes(b[-4:])
    out.append(("trailing bytes", _recrc(trail)))
    big = bytearray(b)
    big[12:16] = _u32(5000)
    out.append(("oversized name", _recrc(bytes(big))))
    name_len = int.from_bytes(b[12:16], "little")
    at = 16 + name_len
    dt = bytearray(b)
    dt[at:at + 4] = _u32(2)
    out.append(("unknown dtype", _recrc(bytes(dt))))
    nd = bytearray(b)
    nd[at + 4:at + 8] = _u32(9)
    out.append(("too many dims", _recrc(bytes(nd))))
    return out
