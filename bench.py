#!/usr/bin/env python
"""Benchmark of the B200 MoE expert path (BASELINE.json configs[1]).

One step = one forward + backward of the OLMoE-1B-7B-shaped MoE layer
(hidden 2048, 64 experts top-8, SwiGLU ffn 1024, 16,384 tokens, bf16) through the
package's CUDA kernels, inputs and weights resident in HBM. The same JSON line
also carries:
  * roofline   - the tcgen05 grouped GEMMs (9 expert GEMMs, 18*RT*H*I FLOP per step)
                 against the measured bf16 peak (MEASURED_PEAKS.json)
  * e2e        - the same metric through b2_moe_fwd_bwd_host(_async) with pinned host
                 x/dout in and out/dx back every step (two-slot copy/compute pipeline)
  * adamw      - the EP-aware sharded AdamW step on the Mula-7B-A1B parameter set
                 (6,919,096,320 params), HBM roofline
  * cpu_baseline - the reference (oracle/_ref, compiled in place) on host cores
`--impl reference` runs only the reference's own CPU implementation of the path.
Multi-GPU (torchrun): each rank runs the layer on its own 16,384 tokens (weak
scaling); the reported time is the max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

H, N, K, I, S = 2048, 64, 8, 1024, 16384
METRIC = "MoE layer fwd+bwd tokens/s"
GEMM_FLOP_PER_TOKEN = 18 * K * H * I          # 9 grouped GEMMs, 2*H*I MACs per routed row
FLOP_PER_TOKEN = GEMM_FLOP_PER_TOKEN + 6 * H * N  # + router fwd/bwd
WORKLOAD = "OLMoE-1B-7B MoE layer: hidden 2048, 64 experts top-8, SwiGLU ffn 1024, 16384 tokens/GPU, bf16"


def env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["hbm_gbs"], p["bf16_tflops"], p.get("bf16_tflops_sustained"), "measured"
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def start(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()

    def _run(self):
        # NVML directly (every 5 ms: a 100 ms timed region gets ~20 samples); nvidia-smi as fallback
        try:
            import pynvml
            pynvml.nvmlInit()
            import torch
            p = torch.cuda.get_device_properties(self.device)  # matched by PCI bus id (visible-device safe)
            h = pynvml.nvmlDeviceGetHandleByPciBusId(f"{p.pci_domain_id:08x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0")
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            bits = [pynvml.nvmlClocksThrottleReasonHwSlowdown, pynvml.nvmlClocksThrottleReasonHwThermalSlowdown,
                    pynvml.nvmlClocksThrottleReasonSwThermalSlowdown, pynvml.nvmlClocksThrottleReasonSwPowerCap]
            while not self._stop.is_set():
                sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                r = pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                self.samples.append([str(sm), str(mx)] + ["Active" if r & b else "Not Active" for b in bits])
                self._stop.wait(0.005)
            return
        except Exception:
            self.samples = []
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                vals = [v.strip() for v in out.stdout.strip().split(",")]
                if len(vals) >= 6:
                    self.samples.append(vals)
            except Exception:
                pass
            self._stop.wait(0.2)

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)
        sm = sorted(float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit())
        mx = max((float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()), default=None)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i].lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "sm_min_mhz": sm[0] if sm else None, "samples": len(self.samples)}


def bind_numa_local(torch, gpu: int):
    """Pin this rank's process to the CPUs closest to its GPU (NVML affinity, matched by PCI
    bus id), so the pinned host buffers of the e2e leg are allocated on the GPU's own NUMA node."""
    try:
        import pynvml
        pynvml.nvmlInit()
        p = torch.cuda.get_device_properties(gpu)
        bus = f"{p.pci_domain_id:08x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
        h = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
        words = pynvml.nvmlDeviceGetCpuAffinity(h, 16)
        cpus = {64 * i + b for i, w in enumerate(words) for b in range(64) if (w >> b) & 1}
        cpus &= set(os.sched_getaffinity(0))
        if cpus:
            os.sched_setaffinity(0, cpus)
            return len(cpus)
    except Exception as e:  # reported, never fatal
        return f"unbound: {type(e).__name__}"
    return "unbound"


# the committed `ncu --set full` capture whose DRAM bytes back roofline.traffic (named, not globbed)
GEMM_TRAFFIC_FILE = os.path.join("profiles", "r02_ncu_gemm_traffic.json")
ADAMW_TRAFFIC_FILE = os.path.join("profiles", "r02_ncu_adamw_traffic.json")
DATASHEET_BF16_TFLOPS = 2250.0  # dense bf16, B200 datasheet


def ncu_traffic():
    """DRAM bytes (read + write) per step of the six expert-GEMM launches, from the committed
    `ncu --set full` capture GEMM_TRAFFIC_FILE (tools/ncu_summary.py writes it)."""
    path = os.path.join(ROOT, GEMM_TRAFFIC_FILE)
    if not os.path.exists(path):
        return None, None
    with open(path) as f:
        d = json.load(f)
    tot = sum(v["dram_bytes"] for k, v in d["kernels"].items()
              if "grouped_gemm_kernel" in k and k.split("<")[1][0] in "012345")
    return tot, GEMM_TRAFFIC_FILE


def cpu_info():
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return model, os.cpu_count() or 1


def ref_ep_threads():
    """the reference runs one thread per EP rank (comm.cpp:90-94): use as many host cores as
    a power-of-two EP width dividing the 64 experts allows"""
    n = min(64, len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1))
    ep = 1
    while ep * 2 <= n:
        ep *= 2
    return ep


def reference_sample(s_local: int, ep: int):
    """fast_moe_forward + fast_moe_backward of the reference (oracle/_ref) at the OLMoE
    shape on an EP world of `ep` rank threads; returns (tokens, seconds)."""
    from oracle import bind  # cpu_baseline / --impl reference leg only
    import ctypes as C
    ref = bind.get("ref") if bind.have_ref() else None
    which = "reference"
    if ref is None:  # the restatement if the reference build is absent
        ref, which = bind.get("orc"), "port"
    cfg = bind.moe_cfg(n_experts=N, top_k=K, hidden=H, intermediate=I, ep=ep, token_block=8)
    sec = C.c_double()
    if which == "reference":
        fn = ref.lib.ref_bench_moe_f32
        fn.argtypes = [C.POINTER(bind.MoeCfg), C.c_int64, C.c_int, C.POINTER(C.c_double)]
        rc = fn(C.byref(cfg), s_local, 1, C.byref(sec))
        if rc != 0:
            raise RuntimeError(ref.lib.ref_last_error())
        return ep * s_local, sec.value, which
    import numpy as np
    router, gate, up, down = ref.expert_weights(cfg, 1234, 0.02)
    x = ref.normal((ep * s_local, H), 77, 0, 1.0)
    t0 = time.perf_counter()
    ref.moe_layer(cfg, s_local, x, router, gate, up, down, x, aux_coeff=0.01)
    return ep * s_local, time.perf_counter() - t0, which


def run_reference_arm(args, rank, world):
    if rank != 0:
        return
    ep = ref_ep_threads()
    s_local = 32
    model, ncpu = cpu_info()
    for _ in range(args.warmup):
        reference_sample(s_local, ep)
    toks, secs = 0, 0.0
    which = "reference"
    for _ in range(args.steps):
        t, s, which = reference_sample(s_local, ep)
        toks += t
        secs += s
    v = toks / secs
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "tokens/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * secs / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": WORKLOAD.replace(", bf16", "") + f" (CPU sample: {ep * s_local} gathered tokens/step, "
                               f"EP={ep} rank threads, f32 - the reference computes in f32)",
                   "parallelism": f"ep{ep} threads (reference World)"},
        "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": ep, "kind": which,
                         "sample": f"fast_moe_forward+backward, OLMoE shape, {ep}x{s_local} tokens per step, "
                                   f"EP={ep} threads on {model} ({ncpu} cpus)"},
        "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def mula_param_set(layers, hid, heads, head_size, inter, experts, vocab, ep=1):
    """ParamSlots of one rank of an MoE preset in Model::param_slots order (model.cpp:189-229):
    (numel, expert?, tp_sharded?); the rank holds experts/ep experts per MoE layer. Pinned to
    the reference's own Model::param_slots / count_params by tests/test_param_set.py."""
    hd = heads * head_size
    nexp = experts // ep
    slots = [(vocab * hid, False, False)]
    for _ in range(layers):
        slots += [(hid, False, False)] + [(hid * hd, False, True)] * 3 + [(hd * hid, False, True)]
        slots += [(hid, False, False), (hid * experts, False, False)] + [(nexp * hid * inter, True, False)] * 3
    slots += [(hid, False, False), (hid * vocab, False, False)]
    return slots


def mula7b_param_set(ep=1):
    """Mula-7B-A1B (preset model.cpp:43-45): 16 layers, hidden 2048, 16 x 128 heads, 64 experts
    of ffn 1024, vocab 50304."""
    return mula_param_set(16, 2048, 16, 128, 1024, 64, 50304, ep)


def bench_adamw(torch, b2, ctx, dev, steps, warmup, world, rank, hbm_peak, dp=1, mode=None):
    """EPSO step on the Mula-7B-A1B set. dp=1: DP=1 x EP=world (the EP axis, strong scaling);
    dp=world: DP=world x EP=1 (the DP axis: every rank holds all experts, expert grads are
    reduce-scattered too — NVLink-bound by construction). mode=SO runs the
    reference's plain sharded optimizer (ShardMode::so, optim.hpp:37) on the same grid: non-expert
    grads all-reduced over EP and every EP rank updates all of them."""
    mode = b2.EPSO if mode is None else mode
    assert sum(n for n, _, _ in mula7b_param_set()) == 6_919_096_320
    per_rank = mula7b_param_set(world // dp)
    total = 6_919_096_320
    gen = torch.Generator(device=dev).manual_seed(11)
    weights = [(torch.randn(n, device=dev, generator=gen, dtype=torch.float32) * 0.02).bfloat16()
               for n, _, _ in per_rank]
    grads = [(torch.randn(n, device=dev, generator=gen, dtype=torch.float32) * 1e-3).bfloat16()
             for n, _, _ in per_rank]
    cfg = b2.AdamWConfig(warmup_steps=0)
    opt = b2.ShardedOptimizer(ctx, cfg, [(w, g, int(e), int(t)) for (w, g, (n, e, t)) in zip(weights, grads, per_rank)],
                              mode)
    for _ in range(warmup):
        opt.step(stats=False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        opt.step(stats=False)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    launches = opt.last_launches()
    st = opt.step(stats=True)
    owned = sum(opt.owned(i)[1] - opt.owned(i)[0] for i in range(len(per_rank)))
    # algorithmic bytes: bf16 grad read twice (norm + update) + fp32 master/m/v r+w + bf16 weight write
    byt = owned * (2 + 2 + 12 + 12 + 2)
    gbs = byt / (ms * 1e-3) / 1e9
    del opt, weights, grads
    torch.cuda.empty_cache()
    ms_t = torch.tensor([ms], device=dev)
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms = float(ms_t.item())
    traffic = None
    tf = os.path.join(ROOT, ADAMW_TRAFFIC_FILE)
    if os.path.exists(tf):  # DRAM bytes per element of the capture (0.5 G elements), scaled to this step
        with open(tf) as f:
            k = json.load(f)["kernels"]
        per_elem = sum(v["dram_bytes"] for v in k.values()) / 0.5e9
        traffic = per_elem * owned
    # NVLink bytes per rank (bf16 reduce-scatter + all-gather) and the roofline time
    # HBM term + NVLink term at ~85 % of 900 GB/s per direction
    ep = world // dp
    exp_el = sum(n for n, e, _ in per_rank if e)
    ne_el = sum(n for n, e, _ in per_rank if not e)
    nvl = 2 * 2 * exp_el * (dp - 1) / dp + 2 * 2 * ne_el * (world - 1) / world
    t_roof = byt / (hbm_peak * 1e9) * 1e3 + nvl / 765e9 * 1e3
    mname = {b2.EPSO: "EPSO", b2.SO: "SO", b2.DDP: "DDP"}[mode]
    return {"metric": f"sharded AdamW step ms ({mname}, Mula-7B-A1B param set, bf16 grads/weights, fp32 state)",
            "parallelism": f"dp{dp} x ep{ep}", "scaling": "strong",
            "nvlink_bytes_per_rank": nvl, "t_roofline_ms": t_roof, "roofline_over_measured": t_roof / ms,
            "ms": ms, "params": total, "owned_params_per_rank": owned, "launches_per_step": launches,
            "grad_norm": st["grad_norm"],
            "roofline": {"bound": "hbm", "achieved": gbs, "peak": hbm_peak, "unit": "GB/s", "frac": gbs / hbm_peak,
                         "traffic": traffic, "traffic_source": ADAMW_TRAFFIC_FILE + " (sumsq + update, per element x owned "
                                                                        "elements)",
                         "algorithmic_bytes_per_step": byt}}


def zipf_tokens(torch, dev, S, Hd, N, s, seed, perm_seed=None):
    """Config E routing (logits[t,e] = log z_e + noise, z_e ∝ (e+1)^-s, identity
    expert permutation, the hottest experts on rank 0) through a router of realistic magnitude:
    x ~ N(1, 1), Wr = column-centred N(0, 1.2825/sqrt(H)) + log z_e / H, so x·Wr = mean(x_t) ·
    log z_e + N(0, 1.28²) (the Gumbel noise's std). Same construction as the parity test
    (tests/test_gpu_bench_shapes.py::zipf_inputs)."""
    g = torch.Generator(device=dev).manual_seed(seed)
    z = (torch.arange(N, device=dev, dtype=torch.float64) + 1.0) ** -s
    z = z / z.sum()
    if perm_seed is not None:  # a seeded expert permutation pi instead of the identity (worst case)
        pg = torch.Generator().manual_seed(perm_seed)
        z = z[torch.randperm(N, generator=pg).to(dev)]
    x = torch.randn((S, Hd), device=dev, generator=g) + 1.0
    wn = torch.randn((Hd, N), device=dev, generator=g, dtype=torch.float64) * (1.2825 / Hd ** 0.5)
    wn -= wn.mean(0, keepdim=True)
    router = (wn + torch.log(z)[None, :] / Hd).float()
    return x.bfloat16(), router.bfloat16()


def bench_zipf(torch, b2, ctx, dev, stream, world, rank, zipf_s, steps, warmup, perm_seed=None):
    """Mula-20B-A2B-shaped layer (H 2048, 96 experts top-8, ffn 1024; model.cpp:46-48) under
    Zipf-skewed routing, EP = world (config E): the load-imbalance stress line."""
    import torch.distributed as dist
    Nz = 96
    cfg = b2.MoeConfig(n_experts=Nz, top_k=K, hidden=H, intermediate=I, ep=world, token_block=8)
    NR = Nz // world
    x, router = zipf_tokens(torch, dev, S, H, Nz, zipf_s, 4242 + rank, perm_seed)
    if world > 1:  # one router for every rank (the tokens differ per rank)
        dist.broadcast(router, src=0)
    gen = torch.Generator(device=dev).manual_seed(99 + rank)
    mk = lambda shape, std: (torch.randn(shape, device=dev, generator=gen) * std).bfloat16()
    gate, up, down, dout = mk((NR, H, I), 0.02), mk((NR, H, I), 0.02), mk((NR, I, H), 0.02), mk((S, H), 1.0)
    layer = b2.MoeLayer(ctx, cfg, torch.bfloat16, S)
    layer.set_graph(True)
    out, apg = torch.empty_like(x), torch.empty((S, Nz), dtype=torch.float32, device=dev)
    grads = dict(input=torch.empty_like(x), router=torch.empty_like(router), gate=torch.empty_like(gate),
                 up=torch.empty_like(up), down=torch.empty_like(down))

    def step():
        layer.forward(x, router, gate, up, down, out=out)
        layer.aux_probs_grad(0.01, out=apg)
        layer.backward(router, gate, up, down, dout, apg, grads=grads)

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = torch.tensor([e0.elapsed_time(e1) / steps], device=dev)
    rows = torch.tensor([float(layer_rt(layer))], device=dev)
    rows_max, rows_sum = rows.clone(), rows.clone()
    if world > 1:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        dist.all_reduce(rows_max, op=dist.ReduceOp.MAX)
        dist.all_reduce(rows_sum, op=dist.ReduceOp.SUM)
    counts = layer.artifacts()["token_counts"]
    del layer
    torch.cuda.empty_cache()
    ms = float(ms.item())
    return {"metric": METRIC + " (Zipf-skewed routing)", "value": world * S / (ms * 1e-3), "unit": "tokens/s",
            "ms_per_step": ms, "zipf_s": zipf_s, "experts": Nz, "ep": world,
            "workload": f"Mula-20B-A2B layer shape: hidden 2048, 96 experts top-8, ffn 1024, {S} tokens/GPU, bf16, "
                        f"Zipf s={zipf_s}, " + ("identity expert permutation" if perm_seed is None
                                                 else f"expert permutation seed {perm_seed}"),
            "rows_per_rank_max_over_mean": float(rows_max.item()) / (float(rows_sum.item()) / world),
            "rank0_rows_per_expert_max_over_mean": float(max(counts)) / max(1e-9, sum(counts) / len(counts))}


def layer_rt(layer):
    """rows routed to this rank's experts in the last step (sum of the expert group sizes)."""
    return int(layer.artifacts()["rt"])


def parity_check(torch, b2, dev, stream, router, gate, up, down, x, dout, world, S_par=256):
    """Post-timing parity of the benchmarked configuration: the first
    S_par tokens of this run's x/dout through a fresh EP=1 layer with this run's weights (the
    full expert set; all-gathered over the EP ranks at N>1), against the CPU oracle
    (oracle/liboracle.so, the C restatement pinned bitwise to the reference) on the same
    bf16 values. Bars (north_star): routing indices and artifacts bit-exact; out / dX within
    2e-2 rel_err elementwise; weight and router grads within 2e-2 of the tensor scale."""
    import numpy as np
    import torch.distributed as dist
    from oracle import bind  # the checker only; the measured path never touches it
    if world > 1:
        full = []
        for w in (gate, up, down):
            buf = torch.empty((w.shape[0] * world,) + tuple(w.shape[1:]), dtype=w.dtype, device=dev)
            dist.all_gather_into_tensor(buf, w.contiguous())
            full.append(buf)
        gate, up, down = full
        if dist.get_rank() != 0:
            return None
    t0 = time.perf_counter()
    Nf = gate.shape[0]
    ctx1 = b2.Context(dev.index, stream=stream)
    cfg = b2.MoeConfig(n_experts=Nf, top_k=K, hidden=H, intermediate=I)
    xs, ds = x[:S_par].contiguous(), dout[:S_par].contiguous()
    layer = b2.MoeLayer(ctx1, cfg, torch.bfloat16, S_par)
    out = layer.forward(xs, router, gate, up, down)
    g = layer.backward(router, gate, up, down, ds, layer.aux_probs_grad(0.01))
    torch.cuda.synchronize()
    _, wts, idx = layer.routing()
    arts = layer.artifacts()
    got = {k: v.float().cpu().numpy() for k, v in g.items()}
    got["out"] = out.float().cpu().numpy()
    layer.close()
    ctx1.close()
    orc = bind.get("orc")
    ocfg = bind.moe_cfg(n_experts=Nf, top_k=K, hidden=H, intermediate=I)
    f = lambda t: t.float().cpu().numpy()
    ref = orc.moe_layer(ocfg, S_par, f(xs), f(router), f(gate), f(up), f(down), f(ds), aux_coeff=0.01)
    oart = orc.artifacts(ocfg, ref["indices"], 0)

    def rel(a, b):
        return float(np.max(np.abs(a.astype(np.float64) - b) / np.maximum(1.0, np.maximum(np.abs(a), np.abs(b)))))

    def scl(a, b):
        return float(np.max(np.abs(a.astype(np.float64) - b)) / max(float(np.max(np.abs(b))), 1e-30))

    art_keys = ("cum_token_counts", "cum_expert_counts", "input_indices", "output_indices", "selected_k")
    res = {"tokens": S_par, "config": f"B dims (H {H}, N {Nf}, K {K}, I {I}), this run's weights and first "
                                      f"{S_par} tokens", "oracle": "oracle/liboracle.so (C restatement, pinned "
                                                                   "bitwise to the reference)",
           "indices_bit_exact": bool(np.array_equal(idx, ref["indices"])),
           "weights_bit_exact": bool(np.array_equal(wts, ref["weights"])),
           "artifacts_bit_exact": bool(all(np.array_equal(np.asarray(arts[k]), oart[k]) for k in art_keys)),
           "out_rel_err": rel(got["out"], ref["out"]), "dx_rel_err": rel(got["input"], ref["dx"]),
           "drouter_scale_err": scl(got["router"], ref["drouter"][0]), "dgate_scale_err": scl(got["gate"], ref["dgate"]),
           "dup_scale_err": scl(got["up"], ref["dup"]), "ddown_scale_err": scl(got["down"], ref["ddown"]),
           "tol": 2e-2}
    res["pass"] = bool(res["indices_bit_exact"] and res["weights_bit_exact"] and res["artifacts_bit_exact"] and
                       all(v <= res["tol"] for k, v in res.items() if k.endswith("_err")))
    res["seconds"] = round(time.perf_counter() - t0, 1)
    return res


def optimizer_cpu_baseline():
    """ShardedOptimizer::step of the reference (oracle/_ref) on the host cores: SO and EPSO at
    DP x EP = 1x1 and 2x2 (the reference's own rank threads), 8 M expert + 8 M non-expert
    elements per rank (SURVEY §8d CPU baseline). ns per logical parameter element per step."""
    from oracle import bind  # cpu_baseline leg only
    import ctypes as C
    if not bind.have_ref():
        return None
    ref = bind.get("ref")
    fn = ref.lib.ref_bench_optim
    fn.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int64, C.c_int64, C.c_int, C.POINTER(C.c_double)]
    ne = nn = 8 << 20
    out = []
    for dp, ep in ((1, 1), (2, 2)):
        for mode, name in ((1, "SO"), (2, "EPSO")):
            sec = C.c_double()
            if fn(dp, ep, mode, ne, nn, 2, C.byref(sec)) != 0:
                raise RuntimeError(ref.lib.ref_last_error())
            logical = ep * ne + nn  # expert elements differ per EP rank; non-expert ones are replicas
            out.append({"mode": name, "dp": dp, "ep": ep, "threads": dp * ep, "step_ms": sec.value * 1e3,
                        "ns_per_element": sec.value * 1e9 / logical, "logical_elements": logical})
    return out


def self_launch(args) -> bool:
    """`bench.py --gpus N` without torchrun: re-launch this script as N ranks (one process per
    GPU, torch.distributed.run over 127.0.0.1) so the JSON line always reports n_gpus = N. The
    rendezvous port is probed free first; a lost race for it (EADDRINUSE) is retried."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ or args.impl == "reference":
        return False
    import random
    import socket
    rc = 1
    for attempt in range(4):
        port = random.randint(20000, 60000)
        with socket.socket() as so:
            try:
                so.bind(("127.0.0.1", port))
            except OSError:
                continue
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
        p = subprocess.run(cmd, stderr=subprocess.PIPE, text=True)
        sys.stderr.write(p.stderr)
        rc = p.returncode
        if rc == 0 or "EADDRINUSE" not in p.stderr and "address already in use" not in p.stderr:
            break
    sys.exit(rc)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--profile", action="store_true", help="print per-stage times to stderr")
    ap.add_argument("--no-adamw", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-parity", action="store_true", help="skip the post-timing oracle check")
    ap.add_argument("--no-graph", action="store_true", help="eager launches instead of CUDA-graph replay")
    ap.add_argument("--zipf", type=float, default=1.2,
                    help="Zipf exponent of the config-E load-imbalance line (96 experts); 0 disables it")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "b200" else args.warmup
    self_launch(args)

    rank, world, local = env_int("RANK", 0), env_int("WORLD_SIZE", 1), env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return

    import torch
    import torch.distributed as dist

    import paper_2604_00785_b200 as b2

    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; refusing to report n_gpus={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    all_cpus = set(os.sched_getaffinity(0))
    numa = bind_numa_local(torch, local)  # host buffers (pinned, first touch) on the GPU's own socket
    # one non-default stream per rank for everything (the layer captures its forward and
    # backward into CUDA graphs on it; the legacy default stream cannot be captured)
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    if world > 1:
        dist.init_process_group("nccl", init_method="env://", device_id=dev)
    hbm_peak, bf16_peak, bf16_sust, peak_kind = measured_peaks()

    # N GPUs = expert parallelism over N ranks (config C): each rank owns N_experts/N experts
    # and its own 16,384 tokens; tokens travel to their experts' ranks by all-to-all
    ep = world
    nccl_id = None
    if world > 1:
        ids = [b2.Context.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(ids, src=0)
        nccl_id = ids[0]
    ctx = b2.Context(local, rank=rank, dp=1, ep=ep, nccl_id=nccl_id, stream=stream)
    cfg = b2.MoeConfig(n_experts=N, top_k=K, hidden=H, intermediate=I, ep=ep, token_block=8)
    NR = N // ep
    gen = torch.Generator(device=dev).manual_seed(1234 + rank)
    mk = lambda shape, std: (torch.randn(shape, device=dev, generator=gen) * std).bfloat16()
    router = (torch.randn((H, N), device=dev, generator=torch.Generator(device=dev).manual_seed(7)) * 0.02).bfloat16()
    gate, up, down = mk((NR, H, I), 0.02), mk((NR, H, I), 0.02), mk((NR, I, H), 0.02)
    x, dout = mk((S, H), 1.0), mk((S, H), 1.0)
    layer = b2.MoeLayer(ctx, cfg, torch.bfloat16, S)
    layer.set_graph(not args.no_graph)
    out = torch.empty_like(x)
    apg = torch.empty((S, N), dtype=torch.float32, device=dev)
    grads = dict(input=torch.empty_like(x), router=torch.empty_like(router), gate=torch.empty_like(gate),
                 up=torch.empty_like(up), down=torch.empty_like(down))

    def step():
        layer.forward(x, router, gate, up, down, out=out)
        nf = layer.last_launches()
        layer.aux_probs_grad(0.01, out=apg)
        layer.backward(router, gate, up, down, dout, apg, grads=grads)
        return nf + 1 + layer.last_launches(), out, grads

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches = 0
    torch.cuda.synchronize()
    t0.record(stream)
    for _ in range(args.steps):
        n, _, _ = step()
        launches += n
    t1.record(stream)
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / args.steps
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    ms_t = torch.tensor([ms], device=dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    value = world * S / (ms_max * 1e-3)

    # per-stage CUDA-event times (same stream as the kernels), separate passes: eager launches
    # (stage_ms) and inside the replayed CUDA graphs (event-record nodes around each stage; the
    # GEMM roofline uses these, the configuration the step time is measured in)
    layer.set_profiling(True)
    for _ in range(args.steps):
        step()
    st = layer.stage_times()
    layer.set_profiling(2)
    for _ in range(2):  # first call eager, second captured
        step()
    st_graph = {k: 0.0 for k in st}
    for _ in range(args.steps):
        step()
        for k_, v in layer.stage_times().items():  # synchronises
            st_graph[k_] += v / args.steps
    layer.set_profiling(False)
    gemm_stages = [k for k in st if k.startswith("gemm")]
    gemm_ms_graph = sum(st_graph[k] for k in gemm_stages)
    graph_pass_ms = sum(st_graph.values())
    gemm_ms_eager = sum(st[k] for k in gemm_stages)
    # the profiled passes run after the timed one, synchronised per step, at the clocks the GPU
    # has settled to by then (power-capped: slower than the timed steps); the GEMMs' SHARE of the
    # profiled in-graph step is applied to the timed step
    gemm_share = gemm_ms_graph / graph_pass_ms
    gemm_ms = gemm_share * ms
    rt = int(layer_rt(layer))
    gemm_flop = 18.0 * rt * H * I
    # expert-parallel load balance: routed rows on this rank vs the mean over ranks
    rows_t = torch.tensor([float(rt)], device=dev)
    rows_max, rows_sum = rows_t.clone(), rows_t.clone()
    if world > 1:
        dist.all_reduce(rows_max, op=dist.ReduceOp.MAX)
        dist.all_reduce(rows_sum, op=dist.ReduceOp.SUM)
    ep_balance = float(rows_max.item()) / (float(rows_sum.item()) / world)
    achieved = gemm_flop / (gemm_ms * 1e-3) / 1e12
    if args.profile and rank == 0:
        for k_, v in st.items():
            print(f"  {k_:>20s} {v:8.3f} ms", file=sys.stderr)
        print(f"  gemm total {gemm_ms:.3f} ms  {achieved:.1f} TFLOP/s  step {ms:.3f} ms  rt {rt}", file=sys.stderr)

    # end to end through the host-buffer entry point (pinned host x/dout in, out/dx back): the
    # pipelined call overlaps step i+1's host->device copies and step i's read-back with compute
    xh, douth = x.cpu().pin_memory(), dout.cpu().pin_memory()
    outh, dxh = torch.empty_like(xh).pin_memory(), torch.empty_like(xh).pin_memory()
    for _ in range(3):
        layer.fwd_bwd_host(xh, douth, router, gate, up, down, outh, dxh, grads, 0.01, wait=False)
    layer.host_wait()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(args.steps):
        layer.fwd_bwd_host(xh, douth, router, gate, up, down, outh, dxh, grads, 0.01, wait=False)
    layer.host_wait()  # every step's results are back in host memory
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = torch.tensor([e0.elapsed_time(e1) / args.steps], device=dev)
    if world > 1:
        dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
    e2e_val = world * S / (float(e2e_ms.item()) * 1e-3)
    tok_bytes = S * H * 2

    del layer
    torch.cuda.empty_cache()
    parity = None
    if not args.no_parity:
        try:
            parity = parity_check(torch, b2, dev, stream, router, gate, up, down, x, dout, world)
        except Exception as e:  # reported in the line, never silently dropped
            parity = {"pass": False, "error": f"{type(e).__name__}: {e}"}
        if world > 1:
            dist.barrier()
    zipf = None
    if args.zipf > 0:
        zipf = bench_zipf(torch, b2, ctx, dev, stream, world, rank, args.zipf, max(2, args.steps // 2), 2)
    adamw = adamw_dp = adamw_so = None
    if not args.no_adamw:
        adamw = bench_adamw(torch, b2, ctx, dev, 5, 2, world, rank, hbm_peak)
        if world > 1:  # the DP axis of config D on its own communicators
            ids = [b2.Context.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(ids, src=0)
            ctx_dp = b2.Context(local, rank=rank, dp=world, ep=1, nccl_id=ids[0], stream=stream)
            adamw_dp = bench_adamw(torch, b2, ctx_dp, dev, 3, 1, world, rank, hbm_peak, dp=world)
            ctx_dp.close()
            adamw_so = bench_adamw(torch, b2, ctx, dev, 3, 1, world, rank, hbm_peak, mode=b2.SO)

    cpu = None
    os.sched_setaffinity(0, all_cpus)  # the CPU reference leg may use every host core
    if rank == 0 and not args.no_cpu:
        try:
            ep = ref_ep_threads()
            toks, secs, which = reference_sample(64, ep)
            model, ncpu = cpu_info()
            cpu = {"value": toks / secs, "unit": "tokens/s", "cores": ep, "kind": which,
                   "sample": f"reference fast_moe_forward+backward at the OLMoE shape, {toks} gathered tokens "
                             f"(EP={ep} rank threads, f32) in {secs:.1f} s on {model} ({ncpu} cpus)"}
        except Exception as e:  # reported, never fatal for the GPU number
            cpu = {"value": None, "unit": "tokens/s", "cores": 0, "kind": "reference", "sample": f"failed: {e}"}
        try:
            cpu["optimizer"] = optimizer_cpu_baseline()
        except Exception as e:
            cpu["optimizer"] = f"failed: {e}"

    traffic, traffic_src = ncu_traffic()
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic (seeded randn tokens, random-init weights)",
            "config": {"workload": WORKLOAD, "global_batch_tokens": world * S,
                       "parallelism": f"ep{world} (dispatch/combine over NVLink peer memory)" if world > 1 else "ep1",
                       "l2": "working set (weights 0.8 GB + activations ~4 GB) >> 126 MB L2; no flush needed",
                       "host_cpus_bound": numa},
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": bf16_peak, "unit": "TFLOP/s",
                         "frac": achieved / bf16_peak, "traffic": traffic, "traffic_source": traffic_src,
                         "traffic_unit": "DRAM bytes per step (6 expert-GEMM launches, ncu --set full)",
                         "peak_kind": peak_kind,
                         "kernel": "tcgen05 grouped GEMMs (6 kinds, 9 expert GEMMs)",
                         "flop_per_step": gemm_flop, "gemm_ms_per_step": gemm_ms,
                         "timing": "gemm_ms_per_step = the six GEMM stages' share of the step, from CUDA events "
                                   "around every stage inside the replayed graphs (separate pass, mean of "
                                   f"{args.steps} steps), times this run's ms_per_step",
                         "gemm_share_of_step": gemm_share, "gemm_ms_graph_pass": gemm_ms_graph,
                         "graph_pass_step_ms": graph_pass_ms, "gemm_ms_eager_pass": gemm_ms_eager,
                         "frac_of_sustained": achieved / bf16_sust if bf16_sust else None,
                         "frac_of_datasheet": achieved / DATASHEET_BF16_TFLOPS},
            "stage_ms": {k: round(v, 4) for k, v in st.items()},
            "stage_ms_graph": {k: round(v, 4) for k, v in st_graph.items()},
            "ep_rows_max_over_mean": ep_balance,
            "model_flop_per_token": FLOP_PER_TOKEN,
            "model_tflops": value * FLOP_PER_TOKEN / 1e12 / world,
            "model_frac_of_measured_peak": value * FLOP_PER_TOKEN / 1e12 / world / bf16_peak,
            "model_frac_of_datasheet": value * FLOP_PER_TOKEN / 1e12 / world / DATASHEET_BF16_TFLOPS,
            "parity": parity,
            "e2e": {"value": e2e_val, "unit": "tokens/s", "h2d_bytes_per_step": 2 * tok_bytes,
                    "d2h_bytes_per_step": 2 * tok_bytes},
            "gpu_launches": launches,
            "clocks": clk,
            "adamw": adamw,
            "adamw_dp_axis": adamw_dp,
            "adamw_so": adamw_so,
            "zipf": zipf,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
