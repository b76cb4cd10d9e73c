"""B200-native MoE expert path and EP-aware sharded AdamW (arxiv 2604.00785 hot path).

Python mirror of the reference operator API over the C-ABI in include/b2moe.h
(libb2moe.so, built in-tree by ``_build.build()``). PyTorch is only the device
memory / stream / process-group plumbing; every computation runs in this
package's CUDA kernels. There is no CPU fallback: importing works anywhere, but
every compute call raises ``B2Error`` (status 3) when no B200 is present, and
``lib()`` raises if the shared library was not built.

Reference API mirrored (file:line under /root/reference/proj):
  MoeConfig             include/optimus/moe.hpp:13-31
  MoeLayer.forward      fast_moe_forward  moe.hpp:344-390
  MoeLayer.backward     fast_moe_backward moe.hpp:392-466
  MoeLayer.aux_probs_grad / aux_loss        moe.hpp:320-342
  MoeLayer.artifacts    RoutingArtifacts  moe.hpp:106-120
  AdamWConfig           include/optimus/optim.hpp:11-25
  ShardedOptimizer      optim.hpp:98-121, src/optim.cpp:109-194
  lr_at_step / shard_slice                  src/optim.cpp:17-50
  memory_report                             src/optim.cpp:196-221
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

PKG = os.path.dirname(os.path.abspath(__file__))
# B2_LIB: an alternative build of the same library for A/B measurements (tools/build_alt.sh)
LIB_PATH = os.environ.get("B2_LIB") or os.path.join(PKG, "libb2moe.so")

F32, BF16 = 0, 1
DDP, SO, EPSO = 0, 1, 2

P = C.c_void_p
I64 = C.c_int64


class B2Error(RuntimeError):
    """Status != 0 from the C-ABI: 1 contract, 2 config, 3 cuda, 4 nccl, 5 io."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"[b2 status {code}] {msg}")
        self.code = code


class ContractError(B2Error):
    pass


class ConfigError(B2Error):
    pass


class IoError(B2Error):
    """optimus::IoError (common.hpp:14-36): unreadable / invalid record files."""


class CMoeCfg(C.Structure):
    _fields_ = [("n_experts", C.c_int64), ("top_k", C.c_int64), ("hidden", C.c_int64),
                ("intermediate", C.c_int64), ("ep", C.c_int32), ("normalize_topk", C.c_int32),
                ("token_block", C.c_int64)]


class CAdamWCfg(C.Structure):
    _fields_ = [("beta1", C.c_double), ("beta2", C.c_double), ("eps", C.c_double),
                ("weight_decay", C.c_double), ("peak_lr", C.c_double), ("min_lr", C.c_double),
                ("warmup_steps", C.c_int64), ("total_steps", C.c_int64), ("clip_norm", C.c_double),
                ("clip_after_warmup_only", C.c_int32), ("round_weights_bf16", C.c_int32)]


class CParam(C.Structure):
    _fields_ = [("weight", P), ("grad", P), ("numel", C.c_int64), ("cls", C.c_int32), ("tp_sharded", C.c_int32)]


class CStepStats(C.Structure):
    _fields_ = [("step", C.c_int64), ("lr", C.c_double), ("grad_norm", C.c_double), ("clip_scale", C.c_double),
                ("nonfinite", C.c_int32)]


# every entry point of include/b2moe.h with its ctypes signature
SIGNATURES = {
    "b2_last_error": (C.c_char_p, []),
    "b2_version": (C.c_char_p, []),
    "b2_device_ok": (C.c_int, []),
    "b2_nccl_unique_id": (C.c_int, [P]),
    "b2_ctx_create": (C.c_int, [C.c_int, P, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, P, P]),
    "b2_ctx_destroy": (C.c_int, [P]),
    "b2_ctx_sync": (C.c_int, [P]),
    "b2_moe_create": (C.c_int, [P, P, C.c_int, I64, P]),
    "b2_moe_destroy": (C.c_int, [P]),
    "b2_moe_forward": (C.c_int, [P, P, P, P, P, P, I64, C.c_int, P]),
    "b2_moe_backward": (C.c_int, [P] + [P] * 11),
    "b2_moe_aux_probs_grad": (C.c_int, [P, C.c_double, P]),
    "b2_moe_aux_loss": (C.c_int, [P, P]),
    "b2_moe_routing": (C.c_int, [P, P, P, P]),
    "b2_moe_artifacts": (C.c_int, [P] + [P] * 11),
    "b2_moe_fwd_bwd_host": (C.c_int, [P, P, P, P, P, P, P, C.c_double, P, P, P, P, P, P, I64]),
    "b2_moe_fwd_bwd_host_async": (C.c_int, [P, P, P, P, P, P, P, C.c_double, P, P, P, P, P, P, I64]),
    "b2_moe_host_wait": (C.c_int, [P]),
    "b2_route": (C.c_int, [P, P, C.c_int, P, P, I64, P, P, P, P]),
    "b2_softmax_topk": (C.c_int, [P, P, I64, I64, I64, C.c_int, P, P, P]),
    "b2_routing_artifacts": (C.c_int, [P, P, P, I64, C.c_int] + [P] * 11),
    "b2_opt_create": (C.c_int, [P, P, P, C.c_int, C.c_int, C.c_int, C.c_int, P]),
    "b2_opt_destroy": (C.c_int, [P]),
    "b2_opt_step": (C.c_int, [P, P]),
    "b2_opt_detect_soft_failure": (C.c_int, [P, C.c_double, C.c_int, P]),
    "b2_opt_state_bytes": (C.c_int64, [P]),
    "b2_opt_owned": (C.c_int, [P, C.c_int, P, P]),
    "b2_opt_get_state": (C.c_int, [P, C.c_int, P, P, P]),
    "b2_opt_gather_state": (C.c_int, [P, C.c_int, P, P, P]),
    "b2_opt_load_state": (C.c_int, [P, C.c_int, P, P, P]),
    "b2_opt_set_step_count": (C.c_int, [P, I64]),
    "b2_adamw_update": (C.c_int, [P, P, P, P, P, C.c_int, I64, C.c_double, I64, P, P, C.c_int, C.c_int]),
    "b2_lr_at_step": (C.c_double, [I64, P]),
    "b2_shard_slice": (C.c_int, [I64, C.c_int, C.c_int, P, P]),
    "b2_memory_report": (C.c_int, [I64, I64, C.c_int, C.c_int, C.c_int, C.c_double, P]),
    "b2_moe_set_profiling": (C.c_int, [P, C.c_int]),
    "b2_moe_set_graph": (C.c_int, [P, C.c_int]),
    "b2_moe_create_ex": (C.c_int, [P, P, C.c_int, I64, P, C.c_int, P]),
    "b2_moe_held_bytes": (I64, [P]),
    "b2_moe_stage_times": (C.c_int, [P, P]),
    "b2_moe_stage_name": (C.c_char_p, [C.c_int]),
    "b2_moe_last_launches": (C.c_int, [P]),
    "b2_opt_last_launches": (C.c_int, [P]),
    "b2_crc32": (C.c_int, [P, P, I64, C.c_uint32, P]),
    "b2_rec_writer_open": (C.c_int, [P, C.c_char_p, P]),
    "b2_rec_writer_add": (C.c_int, [P, C.c_char_p, C.c_int, P, C.c_int, P, C.c_int]),
    "b2_rec_writer_finish": (C.c_int, [P, P, P]),
    "b2_rec_file_open": (C.c_int, [P, C.c_char_p, P]),
    "b2_rec_file_count": (C.c_int, [P, P]),
    "b2_rec_file_info": (C.c_int, [P, C.c_int, P, C.c_int, P, P, P]),
    "b2_rec_file_find": (C.c_int, [P, C.c_char_p, P]),
    "b2_rec_file_read": (C.c_int, [P, C.c_int, I64, I64, P, C.c_int]),
    "b2_rec_file_close": (C.c_int, [P]),
    "b2_opt_write_shard": (C.c_int, [P, C.c_char_p, P, P, P, C.c_int, P, P, P]),
    "b2_opt_restore_shard": (C.c_int, [P, C.c_char_p, P, P, P, C.c_int]),
}

_LIB = None


def lib():
    """The loaded libb2moe.so; raises if it was not built (no fallback exists)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run __graft_entry__.build() (nvcc, sm_100a)")
        lb = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            if os.environ.get("B2_LIB") and not hasattr(lb, name):
                continue  # an A/B build of another revision (tools/ab_build.sh) may predate a symbol
            fn = getattr(lb, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = lb
    return _LIB


def _check(rc: int):
    if rc != 0:
        msg = lib().b2_last_error().decode()
        cls = {1: ContractError, 2: ConfigError, 5: IoError}.get(rc, B2Error)
        raise cls(rc, msg)


def device_ok() -> bool:
    return bool(lib().b2_device_ok())


# ------------------------------------------------------------------ configs

@dataclass
class MoeConfig:
    """optimus::MoeConfig (moe.hpp:13-31) with the reference defaults."""
    n_experts: int = 8
    top_k: int = 2
    hidden: int = 64
    intermediate: int = 128
    ep: int = 1
    token_block: int = 8
    normalize_topk: bool = False

    def c(self) -> CMoeCfg:
        return CMoeCfg(self.n_experts, self.top_k, self.hidden, self.intermediate, self.ep,
                       int(self.normalize_topk), self.token_block)

    def experts_per_rank(self) -> int:
        return self.n_experts // self.ep


@dataclass
class AdamWConfig:
    """optimus::AdamWConfig (optim.hpp:11-25) with the reference defaults."""
    beta1: float = 0.9
    beta2: float = 0.99
    eps: float = 1e-8
    weight_decay: float = 0.1
    peak_lr: float = 4e-4
    min_lr: float = 4e-5
    warmup_steps: int = 2500
    total_steps: int = 100000
    clip_norm: float = 1.0
    clip_after_warmup_only: bool = True
    round_weights_bf16: bool = True

    def c(self) -> CAdamWCfg:
        return CAdamWCfg(self.beta1, self.beta2, self.eps, self.weight_decay, self.peak_lr, self.min_lr,
                         self.warmup_steps, self.total_steps, self.clip_norm, int(self.clip_after_warmup_only),
                         int(self.round_weights_bf16))


def lr_at_step(step: int, cfg: AdamWConfig) -> float:
    c = cfg.c()
    return lib().b2_lr_at_step(step, C.byref(c))


class CMemoryReport(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("weights_bytes", "grads_bytes", "master_bytes", "optim_bytes",
                                          "total_bytes", "capacity_bytes")] + [("feasible", C.c_int32)]


def memory_report(p_expert: int, p_non_expert: int, mode: int, dp: int = 1, ep: int = 1,
                  capacity_gb: float = 64.0) -> dict:
    """memory_report (optim.cpp:196-221); the reference's default capacity (64 GB)."""
    r = CMemoryReport()
    _check(lib().b2_memory_report(p_expert, p_non_expert, mode, dp, ep, capacity_gb, C.byref(r)))
    d = {n: getattr(r, n) for n, _ in CMemoryReport._fields_}
    d["feasible"] = bool(d["feasible"])
    return d


def shard_slice(numel: int, group_size: int, position: int):
    b, e = C.c_int64(), C.c_int64()
    _check(lib().b2_shard_slice(numel, group_size, position, C.byref(b), C.byref(e)))
    return b.value, e.value


# ------------------------------------------------------------------ torch plumbing

def _torch():
    import torch
    return torch


def _dt_code(t) -> int:
    torch = _torch()
    if t.dtype == torch.float32:
        return F32
    if t.dtype == torch.bfloat16:
        return BF16
    raise ContractError(1, f"unsupported dtype {t.dtype} (expected float32 or bfloat16)")


def _ptr(t):
    if t is None:
        return None
    if not t.is_contiguous():
        raise ContractError(1, "tensors must be contiguous")
    return C.c_void_p(t.data_ptr())


class Context:
    """A rank's device + stream (+ NCCL communicators when world > 1): RankCtx (comm.hpp:205-231)."""

    def __init__(self, device: int = 0, rank: int = 0, dp: int = 1, ep: int = 1, tp: int = 1, pp: int = 1,
                 nccl_id: bytes | None = None, stream=None):
        torch = _torch()
        self.device = device
        self.rank, self.dp, self.ep, self.tp, self.pp = rank, dp, ep, tp, pp
        self.world = dp * ep * tp * pp
        torch.cuda.set_device(device)
        self.stream = stream if stream is not None else torch.cuda.current_stream(device)
        h = C.c_void_p()
        idbuf = None if nccl_id is None else (C.c_uint8 * 128).from_buffer_copy(nccl_id)
        _check(lib().b2_ctx_create(device, C.c_void_p(self.stream.cuda_stream), rank, dp, ep, tp, pp,
                                   idbuf, C.byref(h)))
        self.h = h

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        _check(lib().b2_nccl_unique_id(buf))
        return bytes(buf)

    def sync(self):
        _check(lib().b2_ctx_sync(self.h))

    def close(self):
        if self.h:
            _check(lib().b2_ctx_destroy(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class MoeLayer:
    """FastSparseMoE layer on one rank (FastMoeState + fast_moe_forward/backward)."""

    def __init__(self, ctx: Context, cfg: MoeConfig, dtype, max_tokens: int, share_workspace=None,
                 checkpoint: bool = False):
        """share_workspace: another MoeLayer whose activation workspace this one reuses;
        checkpoint: hold only x between forward and backward and replay the forward in
        backward (moe_block_forward's ckpt, blocks.cpp:339-377)."""
        torch = _torch()
        self.ctx, self.cfg = ctx, cfg
        self.dtype = dtype
        self.dt = F32 if dtype == torch.float32 else BF16
        h = C.c_void_p()
        c = cfg.c()
        _check(lib().b2_moe_create_ex(ctx.h, C.byref(c), self.dt, max_tokens,
                                      share_workspace.h if share_workspace is not None else None, int(checkpoint),
                                      C.byref(h)))
        self.h = h
        self._share = share_workspace  # keeps the lender alive
        self.s = 0

    def held_bytes(self) -> int:
        return lib().b2_moe_held_bytes(self.h)

    def forward(self, x, router, gate, up, down, fur: bool = False, out=None):
        torch = _torch()
        if out is None:
            out = torch.empty_like(x)
        self.s = x.shape[0]
        _check(lib().b2_moe_forward(self.h, _ptr(x), _ptr(router), _ptr(gate), _ptr(up), _ptr(down),
                                    x.shape[0], int(fur), _ptr(out)))
        return out

    def backward(self, router, gate, up, down, dout, aux_probs_grad=None, x=None, grads=None):
        """Returns dict(input, router, gate, up, down); `grads` (same keys) supplies the outputs."""
        torch = _torch()
        if grads is None:
            grads = dict(input=torch.empty_like(dout), router=torch.empty_like(router), gate=torch.empty_like(gate),
                         up=torch.empty_like(up), down=torch.empty_like(down))
        _check(lib().b2_moe_backward(self.h, _ptr(router), _ptr(gate), _ptr(up), _ptr(down), _ptr(dout),
                                     _ptr(aux_probs_grad), _ptr(grads["input"]), _ptr(grads["router"]),
                                     _ptr(grads["gate"]), _ptr(grads["up"]), _ptr(grads["down"])))
        return grads

    def aux_probs_grad(self, coeff: float, out=None):
        torch = _torch()
        if out is None:
            out = torch.empty((self.s, self.cfg.n_experts), dtype=torch.float32, device=f"cuda:{self.ctx.device}")
        _check(lib().b2_moe_aux_probs_grad(self.h, coeff, _ptr(out)))
        return out

    def set_graph(self, on: bool = True):
        """CUDA-graph replay of repeated forward/backward calls (needs a non-default stream)."""
        _check(lib().b2_moe_set_graph(self.h, int(on)))

    def aux_loss(self) -> float:
        v = C.c_double()
        _check(lib().b2_moe_aux_loss(self.h, C.byref(v)))
        return v.value

    def routing(self):
        import numpy as np
        S, N, K = self.s, self.cfg.n_experts, self.cfg.top_k
        probs = np.zeros((S, N), np.float32)
        w = np.zeros((S, K), np.float32)
        idx = np.zeros((S, K), np.int64)
        _check(lib().b2_moe_routing(self.h, probs.ctypes.data_as(P), w.ctypes.data_as(P), idx.ctypes.data_as(P)))
        return probs, w, idx

    def artifacts(self):
        return _artifacts_call(lambda *bufs: lib().b2_moe_artifacts(self.h, *bufs), self.cfg,
                               self.s * self.cfg.ep)

    def last_launches(self) -> int:
        return lib().b2_moe_last_launches(self.h)

    NUM_STAGES = 12

    def set_profiling(self, on=True):
        """0 / False off; 1 / True eager per-stage events (mean over calls); 2 per-stage events
        inside the CUDA graphs (graph mode; the last replayed call)."""
        _check(lib().b2_moe_set_profiling(self.h, int(on)))

    def stage_times(self) -> dict:
        import numpy as np
        ms = np.zeros(self.NUM_STAGES, np.float32)
        _check(lib().b2_moe_stage_times(self.h, ms.ctypes.data_as(P)))
        return {lib().b2_moe_stage_name(i).decode(): float(ms[i]) for i in range(self.NUM_STAGES)}

    def fwd_bwd_host(self, x_host, dout_host, router, gate, up, down, out_host, dx_host, grads, aux_coeff=0.0,
                     wait=True):
        """forward+backward with pinned HOST x/dout in and out/dx back (b2_moe_fwd_bwd_host).
        wait=False enqueues on the two-slot copy/compute pipeline and returns
        (b2_moe_fwd_bwd_host_async); results are valid after host_wait()."""
        fn = lib().b2_moe_fwd_bwd_host if wait else lib().b2_moe_fwd_bwd_host_async
        _check(fn(self.h, _ptr(x_host), _ptr(dout_host), _ptr(router), _ptr(gate), _ptr(up), _ptr(down), aux_coeff,
                  _ptr(out_host), _ptr(dx_host), _ptr(grads["router"]), _ptr(grads["gate"]), _ptr(grads["up"]),
                  _ptr(grads["down"]), x_host.shape[0]))

    def host_wait(self):
        _check(lib().b2_moe_host_wait(self.h))

    def close(self):
        if self.h:
            _check(lib().b2_moe_destroy(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _artifacts_call(fn, cfg: MoeConfig, T: int):
    import numpy as np
    NR, K = cfg.experts_per_rank(), cfg.top_k
    TH = (T + cfg.token_block - 1) // cfg.token_block
    cap = max(1, T * K)
    sizes = np.zeros(4, np.int64)
    names = ["token_counts", "partial_token_counts", "partial_cum", "cum_token_counts", "expert_counts",
             "cum_expert_counts", "input_indices", "output_indices", "selected_k", "counter"]
    lens = [NR, max(1, NR * TH), NR * TH + 1, NR + 1, max(1, T), T + 1, cap, cap, cap, max(1, NR * TH)]
    bufs = {n: np.zeros(L, np.int64) for n, L in zip(names, lens)}
    _check(fn(sizes.ctypes.data_as(P), *[bufs[n].ctypes.data_as(P) for n in names]))
    t, th, rt, padded = (int(v) for v in sizes)
    out = dict(t_total=t, th=th, rt=rt, padded_rows=padded)
    for n in names:
        v = bufs[n]
        if n in ("input_indices", "output_indices", "selected_k"):
            v = v[:rt]
        elif n in ("partial_token_counts", "counter"):
            v = v[: NR * th]
        elif n == "expert_counts":
            v = v[:t]
        out[n] = v.copy()
    out["counter"] = out["counter"].reshape(NR, th) if th else out["counter"]
    return out


def route(ctx: Context, cfg: MoeConfig, x, router):
    """route (moe.hpp:58-80) -> logits, probs, weights (fp32), indices (int32)."""
    torch = _torch()
    S, N, K = x.shape[0], cfg.n_experts, cfg.top_k
    dev = x.device
    logits = torch.empty((S, N), dtype=torch.float32, device=dev)
    probs = torch.empty_like(logits)
    w = torch.empty((S, K), dtype=torch.float32, device=dev)
    idx = torch.empty((S, K), dtype=torch.int32, device=dev)
    c = cfg.c()
    _check(lib().b2_route(ctx.h, C.byref(c), _dt_code(x), _ptr(x), _ptr(router), S, _ptr(logits), _ptr(probs),
                          _ptr(w), _ptr(idx)))
    return logits, probs, w, idx


def softmax_topk(ctx: Context, logits, k: int, normalize: bool = False):
    torch = _torch()
    rows, n = logits.shape
    probs = torch.empty_like(logits)
    w = torch.empty((rows, k), dtype=torch.float32, device=logits.device)
    idx = torch.empty((rows, k), dtype=torch.int32, device=logits.device)
    _check(lib().b2_softmax_topk(ctx.h, _ptr(logits), rows, n, k, int(normalize), _ptr(probs), _ptr(w), _ptr(idx)))
    return probs, w, idx


def routing_artifacts(ctx: Context, cfg: MoeConfig, indices, ep_rank: int = 0):
    """count_tokens + generate_indices (moe.hpp:122-197) on a device int32 [T,K] table."""
    c = cfg.c()
    T = indices.shape[0]
    return _artifacts_call(lambda *bufs: lib().b2_routing_artifacts(ctx.h, C.byref(c), _ptr(indices), T, ep_rank,
                                                                    *bufs), cfg, T)


class ShardedOptimizer:
    """EP-aware sharded AdamW (optim.hpp:98-121). params: list of (weight, grad, cls, tp_sharded)."""

    def __init__(self, ctx: Context, cfg: AdamWConfig, params, mode: int = EPSO):
        self.ctx, self.cfg, self.mode = ctx, cfg, mode
        arr = (CParam * len(params))()
        wdt = gdt = None
        for i, (w, g, cls, tps) in enumerate(params):
            arr[i] = CParam(w.data_ptr(), g.data_ptr(), w.numel(), int(cls), int(tps))
            wdt, gdt = _dt_code(w), _dt_code(g)
        self._keep = (arr, params)
        h = C.c_void_p()
        c = cfg.c()
        _check(lib().b2_opt_create(ctx.h, C.byref(c), arr, len(params), mode, wdt, gdt, C.byref(h)))
        self.h = h

    def step(self, stats: bool = True):
        s = CStepStats()
        _check(lib().b2_opt_step(self.h, C.byref(s) if stats else None))
        return dict(step=s.step, lr=s.lr, grad_norm=s.grad_norm, clip_scale=s.clip_scale,
                    nonfinite=bool(s.nonfinite)) if stats else None

    def detect_soft_failure(self, loss: float, node: int = 0) -> int:
        """detect_soft_failure (reliability.cpp:706-723): highest sick node over WORLD, or -1."""
        out = C.c_int()
        _check(lib().b2_opt_detect_soft_failure(self.h, float(loss), int(node), C.byref(out)))
        return out.value

    def state_bytes(self) -> int:
        return lib().b2_opt_state_bytes(self.h)

    def owned(self, p: int):
        b, e = C.c_int64(), C.c_int64()
        _check(lib().b2_opt_owned(self.h, p, C.byref(b), C.byref(e)))
        return b.value, e.value

    def state(self, p: int):
        import numpy as np
        b, e = self.owned(p)
        n = e - b
        ms, m, v = (np.zeros(n, np.float32) for _ in range(3))
        _check(lib().b2_opt_get_state(self.h, p, ms.ctypes.data_as(P), m.ctypes.data_as(P), v.ctypes.data_as(P)))
        return ms, m, v

    def gather_state(self, p: int, numel: int):
        """full (master, exp_avg, exp_avg_sq) of param p over its owning group (collective)."""
        import numpy as np
        ms, m, v = (np.zeros(numel, np.float32) for _ in range(3))
        _check(lib().b2_opt_gather_state(self.h, p, ms.ctypes.data_as(P), m.ctypes.data_as(P), v.ctypes.data_as(P)))
        return ms, m, v

    def load_state(self, p: int, master, exp_avg, exp_avg_sq):
        """restore this rank's owned slice of param p from full fp32 host arrays."""
        import numpy as np
        arrs = [np.ascontiguousarray(a, np.float32) for a in (master, exp_avg, exp_avg_sq)]
        _check(lib().b2_opt_load_state(self.h, p, *[a.ctypes.data_as(P) for a in arrs]))

    def set_step_count(self, n: int):
        _check(lib().b2_opt_set_step_count(self.h, n))

    @staticmethod
    def _shard_args(names, shapes):
        arr = (C.c_char_p * len(names))(*[n.encode() for n in names])
        if shapes is None:
            return arr, None, None
        nd = (C.c_int * len(shapes))(*[len(s) for s in shapes])
        flat = [int(d) for s in shapes for d in s]
        dims = (C.c_int64 * max(len(flat), 1))(*flat)
        return arr, dims, nd

    def write_shard(self, directory: str, names, shapes=None, full: bool = True):
        """write_state_dir's shard file (reliability.cpp:402-460); collective. Returns
        (bytes, crc, model_shard); bytes = crc = 0 on ranks that are not the shard's writer."""
        arr, dims, nd = self._shard_args(names, shapes)
        b, c, m = C.c_int64(), C.c_uint32(), C.c_int()
        _check(lib().b2_opt_write_shard(self.h, directory.encode(), arr, dims, nd, int(full), C.byref(b),
                                        C.byref(c), C.byref(m)))
        return b.value, c.value, m.value

    def restore_shard(self, directory: str, names, shapes=None, full: bool = True):
        """restore_full's per-parameter loop (reliability.cpp:623-675): weights, owned
        master/m/v slices and grads from the shard files; no collective."""
        arr, dims, nd = self._shard_args(names, shapes)
        _check(lib().b2_opt_restore_shard(self.h, directory.encode(), arr, dims, nd, int(full)))

    def last_launches(self) -> int:
        return lib().b2_opt_last_launches(self.h)

    def close(self):
        if self.h:
            _check(lib().b2_opt_destroy(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


REC_F32, REC_BF16 = 0, 1


def crc32(ctx: Context, t, crc: int = 0) -> int:
    """zlib.crc32 of a device tensor's bytes, computed on the GPU (synchronises)."""
    out = C.c_uint32()
    _check(lib().b2_crc32(ctx.h, _ptr(t), t.numel() * t.element_size(), crc, C.byref(out)))
    return out.value


class RecordWriter:
    """RecordFileWriter (reliability.hpp:47-71) over device tensors."""

    def __init__(self, ctx: Context, path: str):
        h = C.c_void_p()
        _check(lib().b2_rec_writer_open(ctx.h, path.encode(), C.byref(h)))
        self.h = h

    def add(self, name: str, t, rec_dtype: int, dims=None):
        dims = list(t.shape) if dims is None else list(dims)
        d = (C.c_int64 * max(len(dims), 1))(*dims)
        _check(lib().b2_rec_writer_add(self.h, name.encode(), rec_dtype, d, len(dims), _ptr(t), _dt_code(t)))

    def add_f32(self, name, t, dims=None):
        self.add(name, t, REC_F32, dims)

    def add_bf16(self, name, t, dims=None):
        self.add(name, t, REC_BF16, dims)

    def finish(self):
        b, c = C.c_int64(), C.c_uint32()
        h, self.h = self.h, None
        _check(lib().b2_rec_writer_finish(h, C.byref(b), C.byref(c)))
        return b.value, c.value


class RecordFile:
    """read_record_file (reliability.cpp:272-320): validated on open; records read into device tensors."""

    def __init__(self, ctx: Context, path: str):
        h = C.c_void_p()
        _check(lib().b2_rec_file_open(ctx.h, path.encode(), C.byref(h)))
        self.h, self.ctx = h, ctx
        n = C.c_int()
        _check(lib().b2_rec_file_count(self.h, C.byref(n)))
        self.records = []
        for i in range(n.value):
            name = C.create_string_buffer(4097)
            dt, nd = C.c_int(), C.c_int()
            dims = (C.c_int64 * 8)()
            _check(lib().b2_rec_file_info(self.h, i, name, 4097, C.byref(dt), dims, C.byref(nd)))
            self.records.append((name.value.decode(), dt.value, tuple(dims[:nd.value])))

    def find(self, name: str) -> int:
        i = C.c_int()
        _check(lib().b2_rec_file_find(self.h, name.encode(), C.byref(i)))
        return i.value

    def read(self, i: int, out, begin: int = 0, end=None):
        """elements [begin, end) of record i into the device tensor out (f32 or bf16)."""
        if end is None:
            end = begin + out.numel()
        _check(lib().b2_rec_file_read(self.h, i, begin, end, _ptr(out), _dt_code(out)))
        return out

    def close(self):
        if self.h:
            _check(lib().b2_rec_file_close(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def adamw_update(ctx: Context, master, exp_avg, exp_avg_sq, grad, lr: float, step: int, cfg: AdamWConfig,
                 weight_out, round_bf16: bool = True):
    """adamw_update (optim.cpp:88-107) on device slices, in place."""
    c = cfg.c()
    _check(lib().b2_adamw_update(ctx.h, _ptr(master), _ptr(exp_avg), _ptr(exp_avg_sq), _ptr(grad), _dt_code(grad),
                                 master.numel(), lr, step, C.byref(c), _ptr(weight_out), _dt_code(weight_out),
                                 int(round_bf16)))
