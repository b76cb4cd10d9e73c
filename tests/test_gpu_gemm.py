"""tcgen05 grouped GEMM kinds in isolation vs a torch fp32 reference of the same op.

Reference ops: grouped_mm / grouped_mm_nt / grouped_mm_weight_grad
(include/optimus/kernels.hpp:111-189) with silu_glu(_backward) (kernels.hpp:262-295)
fused into the epilogues. bf16 operands, fp32 accumulation: tolerance 1e-2 of the
tensor scale (max|d| / max|ref|), written here.

Two shapes: a small one (5 experts, H=320, I=192) and the benchmarked one (config B's
H=2048, I=1024) with a skewed count vector — one expert of more than 16k rows (many
256-row tiles per expert, a 16,900-deep ragged reduction in the weight-gradient kinds),
several empty experts and single-row / exactly-aligned groups.
"""
import ctypes as C

import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

TOL = 1e-2


def _lib():
    import paper_2604_00785_b200 as b2
    lb = b2.lib()
    fn = lb.b2x_grouped_gemm
    fn.restype = C.c_int
    fn.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_int64] + \
        [C.c_void_p] * 12 + [C.c_float]
    return b2, fn


def _p(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def scale_err(got, ref):
    got, ref = got.float(), ref.float()
    return ((got - ref).abs().max() / ref.abs().max().clamp_min(1e-30)).item()


SHAPES = {
    "small": (320, 192, [200, 0, 77, 300, 256]),
    "olmoe": (2048, 1024, [16900, 0, 1, 0, 255, 257, 3000, 0, 512]),
}


@pytest.fixture(scope="module", params=list(SHAPES))
def setup(request):
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    b2, fn = _lib()
    ctx = b2.Context(0)
    torch.manual_seed(0)
    H, I, counts = SHAPES[request.param]
    nr = len(counts)
    starts = [0]
    for c in counts:
        starts.append(starts[-1] + (c + 255) // 256 * 256)
    pmax = starts[-1] + 256
    dev = "cuda"
    ps = torch.tensor(starts, dtype=torch.int32, device=dev)
    cnt = torch.tensor(counts, dtype=torch.int32, device=dev)
    valid = torch.zeros(pmax, dtype=torch.bool, device=dev)
    for e, c in enumerate(counts):
        valid[starts[e]:starts[e] + c] = True

    def rows(shape, s=1.0):
        t = (torch.randn(shape, device=dev) * s)
        t[~valid] = 0
        return t.bfloat16()

    d = dict(b2=b2, fn=fn, ctx=ctx, counts=counts, nr=nr, H=H, I=I, starts=starts, pmax=pmax, ps=ps, cnt=cnt,
             valid=valid)
    d["x"] = rows((pmax, H))
    d["wg"] = (torch.randn(nr, H, I, device=dev) * 0.05).bfloat16()
    d["wu"] = (torch.randn(nr, H, I, device=dev) * 0.05).bfloat16()
    d["wd"] = (torch.randn(nr, I, H, device=dev) * 0.05).bfloat16()
    d["g"] = rows((pmax, I))
    d["u"] = rows((pmax, I))
    d["h"] = rows((pmax, I))
    d["dy"] = rows((pmax, H))
    d["dgu"] = rows((pmax, 2 * I))
    return d


def run(d, kind, out0, out1=None, out2=None, scale=1.0):
    rc = d["fn"](d["ctx"].h, kind, d["H"], d["I"], d["nr"], _p(d["ps"]), _p(d["cnt"]), d["pmax"], _p(d["x"]), _p(d["wg"]),
                 _p(d["wu"]), _p(d["wd"]), _p(d["g"]), _p(d["u"]), _p(d["h"]), _p(d["dy"]), _p(d["dgu"]), _p(out0),
                 _p(out1), _p(out2), scale)
    assert rc == 0, d["b2"].lib().b2_last_error().decode()
    torch.cuda.synchronize()


def groups(d):
    for e in range(d["nr"]):
        yield e, d["starts"][e], d["starts"][e + 1]


def test_fwd_gate_up_swiglu(setup):
    d = setup
    P, I = d["pmax"], d["I"]
    G = torch.full((P, I), 7.0, device="cuda").bfloat16()
    U, Hh = G.clone(), G.clone()
    run(d, 0, G, U, Hh)
    for e, a, b in groups(d):
        if a == b:
            continue
        x = d["x"][a:b].float()
        g_ref = x @ d["wg"][e].float()
        u_ref = x @ d["wu"][e].float()
        assert scale_err(G[a:b], g_ref) < TOL
        assert scale_err(U[a:b], u_ref) < TOL
        h_ref = torch.nn.functional.silu(G[a:b].float()) * U[a:b].float()
        assert scale_err(Hh[a:b], h_ref) < TOL


def test_fwd_down(setup):
    d = setup
    Y = torch.zeros((d["pmax"], d["H"]), device="cuda").bfloat16()
    run(d, 1, Y)
    for e, a, b in groups(d):
        if a == b:
            continue
        assert scale_err(Y[a:b], d["h"][a:b].float() @ d["wd"][e].float()) < TOL


def test_bwd_down_dgrad_swiglu_bwd(setup):
    d = setup
    I = d["I"]
    dgu = torch.zeros((d["pmax"], 2 * I), device="cuda").bfloat16()
    run(d, 2, dgu)
    for e, a, b in groups(d):
        if a == b:
            continue
        dh = d["dy"][a:b].float() @ d["wd"][e].float().t()
        g, u = d["g"][a:b].float(), d["u"][a:b].float()
        s = torch.sigmoid(g)
        du_ref = g * s * dh
        dg_ref = u * dh * (s * (1 + g * (1 - s)))
        assert scale_err(dgu[a:b, :I], dg_ref) < TOL
        assert scale_err(dgu[a:b, I:], du_ref) < TOL


def test_bwd_dx(setup):
    d = setup
    I = d["I"]
    dx = torch.zeros((d["pmax"], d["H"]), device="cuda").bfloat16()
    run(d, 3, dx)
    for e, a, b in groups(d):
        if a == b:
            continue
        ref = d["dgu"][a:b, :I].float() @ d["wg"][e].float().t() + d["dgu"][a:b, I:].float() @ d["wu"][e].float().t()
        assert scale_err(dx[a:b], ref) < TOL


def test_wgrad_down(setup):
    d = setup
    out = torch.full((d["nr"], d["I"], d["H"]), 3.0, device="cuda").bfloat16()
    run(d, 4, out, scale=0.5)
    for e, a, b in groups(d):
        ref = 0.5 * d["h"][a:b].float().t() @ d["dy"][a:b].float()
        if a == b:
            assert out[e].float().abs().max().item() == 0.0  # empty expert -> zero grad
        else:
            assert scale_err(out[e], ref) < TOL


def test_wgrad_gate_up(setup):
    d = setup
    I = d["I"]
    og = torch.full((d["nr"], d["H"], I), 3.0, device="cuda").bfloat16()
    ou = og.clone()
    run(d, 5, og, ou, scale=1.0)
    for e, a, b in groups(d):
        if a == b:
            assert og[e].float().abs().max().item() == 0.0 and ou[e].float().abs().max().item() == 0.0
            continue
        x = d["x"][a:b].float()
        assert scale_err(og[e], x.t() @ d["dgu"][a:b, :I].float()) < TOL
        assert scale_err(ou[e], x.t() @ d["dgu"][a:b, I:].float()) < TOL
