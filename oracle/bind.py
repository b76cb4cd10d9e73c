"""TEST INFRASTRUCTURE ONLY — ctypes bindings to the CPU oracles.

Two libraries share one contract:
  * ``orc`` — oracle/liboracle.so, the C restatement of the reference hot path
    (oracle/moe_oracle.c);
  * ``ref`` — oracle/_ref/libref_optimus.so, the unmodified reference
    (/root/reference/proj) compiled in place with oracle/ref_shim.cpp.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg import this
module. The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORC_PATH = os.path.join(HERE, "liboracle.so")
REF_PATH = os.path.join(HERE, "_ref", "libref_optimus.so")

P = C.c_void_p
I64 = C.c_int64


class MoeCfg(C.Structure):
    _fields_ = [
        ("n_experts", C.c_int64),
        ("top_k", C.c_int64),
        ("hidden", C.c_int64),
        ("intermediate", C.c_int64),
        ("ep", C.c_int32),
        ("normalize_topk", C.c_int32),
        ("token_block", C.c_int64),
    ]


class AdamWCfg(C.Structure):
    _fields_ = [
        ("beta1", C.c_double),
        ("beta2", C.c_double),
        ("eps", C.c_double),
        ("weight_decay", C.c_double),
        ("peak_lr", C.c_double),
        ("min_lr", C.c_double),
        ("warmup_steps", C.c_int64),
        ("total_steps", C.c_int64),
        ("clip_norm", C.c_double),
        ("clip_after_warmup_only", C.c_int32),
        ("round_weights_bf16", C.c_int32),
    ]


def moe_cfg(n_experts=8, top_k=2, hidden=64, intermediate=128, ep=1, token_block=8,
            normalize_topk=False) -> MoeCfg:
    """MoeConfig defaults of the reference (moe.hpp:13-21)."""
    return MoeCfg(n_experts, top_k, hidden, intermediate, ep, int(bool(normalize_topk)), token_block)


def _p(a):
    return None if a is None else a.ctypes.data_as(P)


class Oracle:
    def __init__(self, which: str = "orc"):
        path = ORC_PATH if which == "orc" else REF_PATH
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle library missing: {path} (run make -C oracle)")
        self.which = which
        self.pre = "orc_" if which == "orc" else "ref_"
        self.lib = C.CDLL(path)
        f = self._f
        f("last_error").restype = C.c_char_p
        f("lr_at_step").restype = C.c_double
        f("lr_at_step").argtypes = [I64, C.POINTER(AdamWCfg)]
        f("normal_init_f32").argtypes = [P, I64, C.c_uint64, C.c_uint64, C.c_double]
        f("fnv1a").restype = C.c_uint64
        f("fnv1a").argtypes = [C.c_char_p]
        f("hash_mix").restype = C.c_uint64
        f("hash_mix").argtypes = [C.c_uint64, C.c_uint64]
        f("bf16_round").restype = C.c_float
        f("bf16_round").argtypes = [C.c_float]
        f("adamw_update").argtypes = [P, P, P, P, I64, C.c_double, I64, C.POINTER(AdamWCfg), P, C.c_int]
        f("moe_layer_f32").argtypes = [C.POINTER(MoeCfg), I64] + [P] * 6 + [C.c_int, C.c_double, C.c_int] + [P] * 10
        f("moe_layer_f64").argtypes = f("moe_layer_f32").argtypes
        f("sharded_steps").argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(AdamWCfg), C.c_int,
                                       P, P, P, P, P, C.c_int, P, P, P, P, P, P, P]

    def _f(self, name):
        return getattr(self.lib, self.pre + name)

    def _check(self, rc):
        if rc != 0:
            raise RuntimeError(f"{self.which}: rc={rc}: {self._f('last_error')().decode()}")

    # ---- generators (common.hpp:83-87, kernels.hpp:392-399) ----
    def normal(self, shape, seed, tag=0, std=1.0):
        out = np.empty(int(np.prod(shape)), np.float32)
        self._f("normal_init_f32")(_p(out), out.size, seed, tag, std)
        return out.reshape(shape)

    def fnv1a(self, s: str) -> int:
        return self._f("fnv1a")(s.encode())

    def hash_mix(self, a, b) -> int:
        return self._f("hash_mix")(a, b)

    def expert_weights(self, cfg: MoeCfg, seed=1234, std=0.02):
        """init_expert_weights (moe.hpp:500-523), full logical expert set."""
        H, N, I = cfg.hidden, cfg.n_experts, cfg.intermediate
        router = self.normal((H, N), seed, self.fnv1a("moe.router"), std)
        gate = self.normal((N, H, I), seed, self.fnv1a("moe.gate"), std)
        up = self.normal((N, H, I), seed, self.fnv1a("moe.up"), std)
        down = self.normal((N, I, H), seed, self.fnv1a("moe.down"), std)
        return router, gate, up, down

    # ---- routing ----
    def route(self, cfg: MoeCfg, x):
        x = np.ascontiguousarray(x, np.float32)
        S = x.shape[0]
        N, K = cfg.n_experts, cfg.top_k
        logits = np.empty((S, N), np.float32)
        probs = np.empty((S, N), np.float32)
        w = np.empty((S, K), np.float32)
        idx = np.empty((S, K), np.int64)
        return logits, probs, w, idx

    def route_f32(self, cfg: MoeCfg, x, router):
        x = np.ascontiguousarray(x, np.float32)
        router = np.ascontiguousarray(router, np.float32)
        logits, probs, w, idx = self.route(cfg, x)
        self._check(self._f("route_f32")(C.byref(cfg), I64(x.shape[0]), _p(x), _p(router), _p(logits),
                                         _p(probs), _p(w), _p(idx)))
        return logits, probs, w, idx

    def softmax_topk(self, logits, k):
        logits = np.ascontiguousarray(logits, np.float32)
        rows, n = logits.shape
        probs = np.empty_like(logits)
        vals = np.empty((rows, k), np.float32)
        idx = np.empty((rows, k), np.int64)
        self._check(self._f("softmax_topk_f32")(I64(rows), I64(n), I64(k), _p(logits), _p(probs), _p(vals),
                                                _p(idx)))
        return probs, vals, idx

    def artifacts(self, cfg: MoeCfg, indices, ep_rank=0):
        """count_tokens + generate_indices (moe.hpp:122-197)."""
        indices = np.ascontiguousarray(indices, np.int64)
        T, K = indices.shape
        NR = cfg.n_experts // cfg.ep
        TH = (T + cfg.token_block - 1) // cfg.token_block
        cap = max(1, T * K)
        sizes = np.zeros(2, np.int64)
        bufs = dict(
            token_counts=np.zeros(NR, np.int64),
            partial_token_counts=np.zeros(max(1, NR * TH), np.int64),
            partial_cum=np.zeros(NR * TH + 1, np.int64),
            cum_token_counts=np.zeros(NR + 1, np.int64),
            expert_counts=np.zeros(max(1, T), np.int64),
            cum_expert_counts=np.zeros(T + 1, np.int64),
            input_indices=np.zeros(cap, np.int64),
            output_indices=np.zeros(cap, np.int64),
            selected_k=np.zeros(cap, np.int64),
            counter=np.zeros(max(1, NR * TH), np.int64),
        )
        rc = self._f("routing_artifacts")(C.byref(cfg), I64(T), _p(indices), C.c_int(ep_rank), _p(sizes),
                                          *[_p(b) for b in bufs.values()])
        self._check(rc)
        th, rt = int(sizes[0]), int(sizes[1])
        out = dict(th=th, rt=rt, t_total=T)
        for k_, v in bufs.items():
            if k_ in ("input_indices", "output_indices", "selected_k"):
                out[k_] = v[:rt].copy()
            elif k_ in ("partial_token_counts", "counter"):
                out[k_] = v[: NR * th].copy()
            elif k_ == "expert_counts":
                out[k_] = v[:T].copy()
            else:
                out[k_] = v.copy()
        out["counter"] = out["counter"].reshape(NR, th) if th else out["counter"]
        return out

    # ---- full layer ----
    def moe_layer(self, cfg: MoeCfg, s_local, x, router, gate, up, down, dout=None, fur=False,
                  aux_coeff=0.0, dtype=np.float32):
        """fast_moe_forward (+ backward when dout is given) over an EP world of cfg.ep
        ranks; full logical tensors in/out (see ref_shim.cpp)."""
        E = cfg.ep
        H, I, N, K = cfg.hidden, cfg.intermediate, cfg.n_experts, cfg.top_k
        cv = lambda a: np.ascontiguousarray(a, dtype)
        x, router, gate, up, down = map(cv, (x, router, gate, up, down))
        bwd = dout is not None
        dout = cv(dout) if bwd else np.zeros_like(x)
        T = E * s_local
        r = dict(out=np.zeros((T, H), dtype), dx=np.zeros((T, H), dtype), drouter=np.zeros((E, H, N), dtype),
                 dgate=np.zeros((N, H, I), dtype), dup=np.zeros((N, H, I), dtype), ddown=np.zeros((N, I, H), dtype),
                 weights=np.zeros((T, K), dtype), indices=np.zeros((T, K), np.int64),
                 probs=np.zeros((T, N), dtype), aux=np.zeros(E, np.float64))
        fn = self._f("moe_layer_f32" if dtype == np.float32 else "moe_layer_f64")
        rc = fn(C.byref(cfg), I64(s_local), _p(x), _p(router), _p(gate), _p(up), _p(down), _p(dout),
                C.c_int(int(fur)), C.c_double(aux_coeff), C.c_int(int(bwd)),
                _p(r["out"]), _p(r["dx"]), _p(r["drouter"]), _p(r["dgate"]), _p(r["dup"]), _p(r["ddown"]),
                _p(r["weights"]), _p(r["indices"]), _p(r["probs"]), _p(r["aux"]))
        self._check(rc)
        return r

    def dense_moe_forward(self, cfg: MoeCfg, x, gate, up, down, weights, indices):
        """reference_moe_forward (moe.hpp:471-497): the dense per-token oracle, full expert set."""
        cv = lambda a: np.ascontiguousarray(a, np.float32)
        x, gate, up, down, weights = map(cv, (x, gate, up, down, weights))
        indices = np.ascontiguousarray(indices, np.int64)
        out = np.zeros_like(x)
        self._check(self._f("dense_moe_forward_f32")(C.byref(cfg), I64(x.shape[0]), _p(x), _p(gate), _p(up),
                                                     _p(down), _p(weights), _p(indices), _p(out)))
        return out

    # ---- optimizer ----
    def adamw_cfg(self, **kw) -> AdamWCfg:
        c = AdamWCfg()
        self._f("adamw_default_cfg")(C.byref(c))
        for k_, v in kw.items():
            setattr(c, k_, v)
        return c

    def lr_at_step(self, step, cfg: AdamWCfg):
        return self._f("lr_at_step")(I64(step), C.byref(cfg))

    def memory_report(self, p_expert, p_non_expert, mode, dp=1, ep=1, capacity_gb=64.0):
        """memory_report (optim.cpp:196-221)."""
        out = np.zeros(7, np.float64)
        f = self._f("memory_report")
        f.argtypes = [I64, I64, C.c_int, C.c_int, C.c_int, C.c_double, P]
        self._check(f(p_expert, p_non_expert, mode, dp, ep, capacity_gb, _p(out)))
        keys = ("weights_bytes", "grads_bytes", "master_bytes", "optim_bytes", "total_bytes", "capacity_bytes")
        d = {k: float(v) for k, v in zip(keys, out)}
        d["feasible"] = bool(out[6])
        return d

    def shard_slice(self, numel, g, pos):
        b, e = I64(), I64()
        self._check(self._f("shard_slice")(I64(numel), C.c_int(g), C.c_int(pos), C.byref(b), C.byref(e)))
        return b.value, e.value

    def adamw_update(self, master, m, v, grad, lr, step, cfg: AdamWCfg, round_bf16=True):
        master, m, v = master.copy(), m.copy(), v.copy()
        grad = np.ascontiguousarray(grad, np.float32)
        out = np.empty_like(master)
        self._check(self._f("adamw_update")(_p(master), _p(m), _p(v), _p(grad), I64(master.size),
                                            C.c_double(lr), I64(step), C.byref(cfg), _p(out),
                                            C.c_int(int(round_bf16))))
        return master, m, v, out

    def sharded_steps(self, dp, ep, tp, mode, cfg: AdamWCfg, numel, cls, tp_sharded, w_init, grads):
        """ShardedOptimizer over a dp x ep x tp world (mode 0 ddp, 1 so, 2 epso).
        w_init [W, total]; grads [steps, W, total]."""
        W = dp * ep * tp
        numel = np.asarray(numel, np.int64)
        cls = np.asarray(cls, np.int32)
        tps = np.asarray(tp_sharded, np.int32)
        total = int(numel.sum())
        w_init = np.ascontiguousarray(w_init, np.float32).reshape(W, total)
        grads = np.ascontiguousarray(grads, np.float32)
        steps = grads.shape[0]
        w_out = np.zeros((W, total), np.float32)
        master = np.zeros((W, total), np.float32)
        m = np.zeros((W, total), np.float32)
        v = np.zeros((W, total), np.float32)
        owned = np.zeros((W, len(numel), 2), np.int64)
        stats = np.zeros((steps, W, 3), np.float64)
        sb = np.zeros(W, np.int64)
        self._check(self._f("sharded_steps")(dp, ep, tp, mode, C.byref(cfg), len(numel), _p(numel), _p(cls),
                                             _p(tps), _p(w_init), _p(grads), steps, _p(w_out), _p(master), _p(m),
                                             _p(v), _p(owned), _p(stats), _p(sb)))
        return dict(weights=w_out, master=master, m=m, v=v, owned=owned, stats=stats, state_bytes=sb)


    # ---- record files (reliability.hpp:33-70, reliability.cpp:222-320) ----
    def record_file_write(self, path, records):
        """records: [(name, rec_dtype 0|1, dims, f32 array)] -> (bytes, crc) of the file at path."""
        names = b"".join(n.encode() + b"\0" for n, _, _, _ in records)
        dts = np.array([d for _, d, _, _ in records], np.int32)
        nds = np.array([len(s) for _, _, s, _ in records], np.int32)
        dims = np.array([x for _, _, s, _ in records for x in s] or [0], np.int64)
        data = np.concatenate([np.asarray(a, np.float32).ravel() for *_, a in records] or
                              [np.zeros(1, np.float32)])
        n = len(records)
        if self.which == "orc":
            f = self._f("record_file_bytes")
            f.restype = I64
            args = (n, names, _p(dts), _p(nds), _p(dims), _p(data))
            size = f(*args, None)
            if size < 0:
                self._check(1)
            out = np.zeros(size, np.uint8)
            f(*args, _p(out))
            with open(path, "wb") as fh:
                fh.write(out.tobytes())
            return int(size), int.from_bytes(out[-4:].tobytes(), "little")
        b, c = I64(), C.c_uint32()
        self._check(self._f("record_file_write")(path.encode(), n, names, _p(dts), _p(nds), _p(dims), _p(data),
                                                 C.byref(b), C.byref(c)))
        return b.value, c.value

    def record_file_read(self, path):
        """read_record_file -> (count, all records widened to f32 and concatenated);
        raises RuntimeError with the reference's message on an invalid file."""
        cnt, tot = I64(), I64()
        if self.which == "orc":
            raw = np.fromfile(path, np.uint8)
            f = self._f("record_file_parse")
            self._check(f(_p(raw), I64(raw.size), C.byref(cnt), C.byref(tot), None, I64(0)))
            out = np.zeros(max(tot.value, 1), np.float32)
            self._check(f(_p(raw), I64(raw.size), C.byref(cnt), C.byref(tot), _p(out), I64(out.size)))
        else:
            f = self._f("record_file_read")
            self._check(f(path.encode(), C.byref(cnt), C.byref(tot), None, I64(0)))
            out = np.zeros(max(tot.value, 1), np.float32)
            self._check(f(path.encode(), C.byref(cnt), C.byref(tot), _p(out), I64(out.size)))
        return cnt.value, out[:tot.value]

    # ---- the model's parameter set (reference only: src/model.cpp:31-91, 189-229) ----
    def count_params(self, preset: str):
        tot, act = I64(), I64()
        self._check(self._f("count_params")(preset.encode(), C.byref(tot), C.byref(act)))
        return tot.value, act.value

    def param_slots(self, preset: str, ep: int = 1, ep_coord: int = 0):
        """Model::param_slots of one rank: list of (numel, expert?, tp_sharded?) in slot order."""
        cap = 4096
        numel, ex, tp = np.zeros(cap, np.int64), np.zeros(cap, np.int32), np.zeros(cap, np.int32)
        n = C.c_int()
        self._check(self._f("param_slots")(preset.encode(), ep, ep_coord, _p(numel), _p(ex), _p(tp), cap,
                                           C.byref(n)))
        return [(int(numel[i]), bool(ex[i]), bool(tp[i])) for i in range(min(n.value, cap))]


_CACHE: dict = {}


def get(which="orc") -> Oracle:
    if which not in _CACHE:
        _CACHE[which] = Oracle(which)
    return _CACHE[which]


def have_ref() -> bool:
    return os.path.exists(REF_PATH)
