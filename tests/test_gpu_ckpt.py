"""GPU parity of the sharded-checkpoint record files through the C-ABI:

* b2_crc32 (GPU crc32 over HBM) equals zlib.crc32 on ragged sizes, unaligned pointers and
  chained seeds;
* b2_rec_writer_* over device tensors writes files byte-identical to the reference's
  RecordFileWriter (the committed golden files, tests/golden/records_*.bin, and the
  oracle restatement for larger multi-chunk payloads);
* b2_rec_file_* validates like read_record_file (same message per corruption class) and
  reads any element range back into f32 / bf16 device memory;
* b2_opt_write_shard / b2_opt_restore_shard: the shard file parses under the oracle with
  the gathered state, and a restored optimizer steps bitwise like the original.
Bars: bitwise everywhere (integer / byte work)."""
import os
import zlib

import numpy as np
import pytest

import record_cases
from test_records import WANT

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def b2ctx():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2604_00785_b200 as b2
    return b2, b2.Context(0)


@pytest.mark.parametrize("n", [0, 1, 15, 16, 17, 511, 512, 513, 4096, 65535, 65536, 65537, 1_000_003,
                               (32 << 20) + 12345])
@pytest.mark.parametrize("offset", [0, 3])
def test_crc32_matches_zlib(b2ctx, n, offset):
    b2, ctx = b2ctx
    g = torch.Generator(device="cuda").manual_seed(n + offset)
    buf = torch.randint(0, 256, (n + offset,), dtype=torch.uint8, device="cuda", generator=g)
    view = buf[offset:]
    host = view.cpu().numpy().tobytes()
    assert b2.crc32(ctx, view) == zlib.crc32(host)
    # continuation from a seed equals zlib's chained crc
    assert b2.crc32(ctx, view, 0x12345678) == zlib.crc32(host, 0x12345678)


def bf16_bits(a):
    """f32_to_bf16_bits (common.hpp:116-122) in numpy: NaN stays quiet, else RNE"""
    u = np.ascontiguousarray(a, np.float32).ravel().view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) & 0xFFFF
    nan = np.isnan(np.asarray(a, np.float32).ravel())
    r[nan] = (u[nan] >> 16) | 0x40
    return r.astype(np.uint16)


def widen(bits):
    return (bits.astype(np.uint32) << 16).view(np.float32)


@pytest.mark.parametrize("case", ["roundtrip", "rounding", "empty", "corrupt_base", "mixed"])
@pytest.mark.parametrize("src", ["f32", "bf16"])
def test_writer_matches_reference_golden(b2ctx, orc, tmp_path, case, src):
    b2, ctx = b2ctx
    recs = record_cases.cases(orc)[case]
    path = str(tmp_path / "w.bin")
    w = b2.RecordWriter(ctx, path)
    for name, dt, dims, a in recs:
        t = torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda()
        if src == "bf16" and dt == 1:  # bf16 sources: device tensors already in bf16 (our weights / grads)
            t = torch.from_numpy(bf16_bits(a).view(np.int16)).cuda().view(torch.bfloat16)
        w.add(name, t.reshape(-1), dt, dims)
    nbytes, crc = w.finish()
    got = open(path, "rb").read()
    gold = open(os.path.join(GOLD, f"records_{case}.bin"), "rb").read()
    assert got == gold
    assert nbytes == len(gold) and crc == zlib.crc32(gold[:-4])


def test_reader_records_and_ranges(b2ctx, orc):
    b2, ctx = b2ctx
    recs = record_cases.cases(orc)["mixed"]
    f = b2.RecordFile(ctx, os.path.join(GOLD, "records_mixed.bin"))
    assert [(n, d, tuple(s)) for n, d, s, _ in recs] == f.records
    for i, (name, dt, dims, a) in enumerate(recs):
        assert f.find(name) == i
        a = np.asarray(a, np.float32).ravel()
        want = a if dt == 0 else widen(bf16_bits(a))
        out = torch.full((a.size,), 7.0, device="cuda")
        f.read(i, out)
        assert np.array_equal(out.cpu().numpy().view(np.uint32), want.view(np.uint32)), name
        if a.size >= 4:  # a sub-range, into bf16 device memory
            o16 = torch.zeros(a.size - 3, dtype=torch.bfloat16, device="cuda")
            f.read(i, o16, 2, a.size - 1)
            wb = bf16_bits(want[2:a.size - 1]).view(np.int16)
            assert np.array_equal(o16.cpu().view(torch.int16).numpy(), wb), name
    assert f.find("absent") == -1
    f.close()


def test_reader_rejects_corruptions_like_the_reference(b2ctx, tmp_path):
    b2, ctx = b2ctx
    good = open(os.path.join(GOLD, "records_corrupt_base.bin"), "rb").read()
    path = str(tmp_path / "c.bin")
    for what, data in record_cases.corruptions(good):
        with open(path, "wb") as fh:
            fh.write(data)
        with pytest.raises(b2.IoError) as e:
            b2.RecordFile(ctx, path)
        assert str(e.value).endswith(path + ": " + WANT[what]), (what, str(e.value))
    with pytest.raises(b2.IoError):
        b2.RecordFile(ctx, str(tmp_path / "missing.bin"))


def test_large_multichunk_round_trip(b2ctx, orc, tmp_path):
    """payloads spanning several 32 MB streaming chunks and 64 KB crc segments, ragged ends"""
    b2, ctx = b2ctx
    g = torch.Generator(device="cuda").manual_seed(5)
    a = torch.randn(20_000_017, device="cuda", generator=g)            # 80 MB f32
    b = torch.randn(33_554_437, device="cuda", generator=g).bfloat16()  # 64 MB bf16
    path = str(tmp_path / "big.bin")
    w = b2.RecordWriter(ctx, path)
    w.add_f32("a", a)
    w.add_bf16("a16", a)   # f32 source, rounded on the GPU
    w.add_bf16("b", b, (33_554_437,))
    nbytes, crc = w.finish()
    raw = np.fromfile(path, np.uint8)
    assert nbytes == raw.size and crc == zlib.crc32(raw[:-4].tobytes())
    cnt, vals = orc.record_file_read(path)  # the oracle's read_record_file accepts it
    assert cnt == 3
    ah = a.cpu()
    n = a.numel()
    assert np.array_equal(vals[:n].view(np.uint32), ah.numpy().view(np.uint32))
    assert torch.equal(torch.from_numpy(vals[n:2 * n]).view(torch.int32), ah.bfloat16().float().view(torch.int32))
    assert torch.equal(torch.from_numpy(vals[2 * n:]).view(torch.int32), b.cpu().float().view(torch.int32))
    f = b2.RecordFile(ctx, path)
    out = torch.empty(n - 1000, device="cuda")
    f.read(0, out, 1000, n)
    assert torch.equal(out, a[1000:])
    ob = torch.empty_like(b)
    f.read(2, ob)
    assert torch.equal(ob.view(torch.int16), b.view(torch.int16))


NUMEL = [33, 130_001, 7, 4096]
CLS = [0, 1, 0, 1]
SHAPES = [(3, 11), (130_001,), (7,), (64, 64)]


@pytest.mark.parametrize("mode", [0, 1, 2], ids=["ddp", "so", "epso"])
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32], ids=["bf16", "f32"])
def test_optimizer_shard_round_trip(b2ctx, orc, tmp_path, mode, dtype):
    b2, ctx = b2ctx
    total = sum(NUMEL)
    rng = np.random.default_rng(mode)
    w0 = torch.from_numpy((rng.standard_normal(total) * 0.05).astype(np.float32)).to(dtype).cuda()
    cfg = b2.AdamWConfig(warmup_steps=1, total_steps=20)

    def build(W, G):
        ps, off = [], 0
        for n, c in zip(NUMEL, CLS):
            ps.append((W[off:off + n], G[off:off + n], c, 0))
            off += n
        return b2.ShardedOptimizer(ctx, cfg, ps, mode)

    W, G = w0.clone(), torch.zeros(total, dtype=dtype, device="cuda")
    opt = build(W, G)
    for s in range(3):
        G.copy_(torch.from_numpy((rng.standard_normal(total) * 0.01).astype(np.float32)).to(dtype))
        opt.step(stats=False)
    torch.cuda.synchronize()
    names = [f"layers.0.p{p}" for p in range(len(NUMEL))]
    nbytes, crc, shard = opt.write_shard(str(tmp_path), names, SHAPES)
    path = str(tmp_path / f"shard-{shard}.bin")
    assert shard == 0 and nbytes == os.path.getsize(path)
    # the oracle's read_record_file: record order and payloads of write_state_dir
    cnt, vals = orc.record_file_read(path)
    assert cnt == 5 * len(NUMEL)
    f = b2.RecordFile(ctx, path)
    want_names = [f"{n}{sfx}" for n in names for sfx in (".w16", ".master", ".m", ".v", ".g16")]
    assert [r[0] for r in f.records] == want_names
    assert [r[2] for r in f.records][::5] == [tuple(s) for s in SHAPES]
    at, off = 0, 0
    for p, n in enumerate(NUMEL):
        full = opt.gather_state(p, n)
        w16 = W[off:off + n].float().bfloat16().float().cpu().numpy()
        g16 = G[off:off + n].float().bfloat16().float().cpu().numpy()
        for arr in (w16, *full, g16):
            assert np.array_equal(vals[at:at + n].view(np.uint32), np.asarray(arr, np.float32).view(np.uint32))
            at += n
        off += n
    f.close()
    # restore into a fresh optimizer; one more identical step on both is bitwise equal
    W2, G2 = torch.zeros_like(W), torch.zeros_like(G)
    opt2 = build(W2, G2)
    opt2.restore_shard(str(tmp_path), names, SHAPES)
    opt2.set_step_count(3)
    torch.cuda.synchronize()
    if dtype == torch.bfloat16:
        assert torch.equal(W2.view(torch.int16), W.view(torch.int16))
        assert torch.equal(G2.view(torch.int16), G.view(torch.int16))
    else:  # f32 weights are bf16-representable after a rounded step; grads come back bf16-rounded
        assert torch.equal(W2, W)
        assert torch.equal(G2, G.bfloat16().float())
        G.copy_(G2)
    for p in range(len(NUMEL)):
        for a, b in zip(opt.state(p), opt2.state(p)):
            assert np.array_equal(a, b)
    opt.step(stats=False)
    opt2.step(stats=False)
    torch.cuda.synchronize()
    assert torch.equal(W2.float(), W.float())
    for p in range(len(NUMEL)):
        for a, b in zip(opt.state(p), opt2.state(p)):
            assert np.array_equal(a, b)
    # weights-only files (write_model_only): .w16 records alone
    d2 = tmp_path / "model"
    d2.mkdir()
    nb2, _, _ = opt.write_shard(str(d2), names, SHAPES, full=False)
    f2 = b2.RecordFile(ctx, str(d2 / "shard-0.bin"))
    assert [r[0] for r in f2.records] == [n + ".w16" for n in names]
    f2.close()
    # a wrong shape is a contract error, a missing record an io error
    with pytest.raises(b2.ContractError):
        opt2.restore_shard(str(tmp_path), names, [(33,), (130_001,), (7,), (4096,)])
    with pytest.raises(b2.IoError):
        opt2.restore_shard(str(tmp_path), [n + "x" for n in names], SHAPES)
    opt.close()
    opt2.close()
