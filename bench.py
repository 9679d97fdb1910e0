#!/usr/bin/env python
"""bench.py -- MiniKV attention hot path on B200 (one JSON line on rank 0).

Headline workload (BASELINE.json configs[1]): Llama-3-8B-shaped GQA decode
(32 q / 8 kv heads, d = 128, 32 layers, pyramid budget, 20% = 10% HH + 10% RW of
a 32K context), batch 16 per GPU.  A "step" = one decode step through all 32
layers: per layer decode_append (+ n_r flush) and 2-bit attention over
[pages ; residual] for 16 x 8 (seq, kv-head) units (K4).  ``value`` is
whole-job decode tokens/s with inputs resident in HBM; ``e2e`` is the same
through the C-ABI with host (pinned) buffers copied in and out every step.
A ``prefill`` object reports the selective-FA prefill (K1) TFLOP/s on the
Mistral-7B-shaped layer of configs[3] when the kernel is available.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl mkv|reference]

N > 1 runs under torch.distributed.run, one rank per GPU, each rank an
independent batch-16 shard (weak scaling; the attention path has no exchange).
``--impl reference`` times the reference CPU implementation (oracle/_ref, the
unmodified reference sources) on this host's cores, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "2-bit-KV decode attn tokens/s (Llama-3-8B GQA, 32K ctx, 20% pyramid budget)"
UNIT = "tokens/s"
SEED = 2024

CFG = dict(batch=16, layers=32, n_q_heads=32, n_kv_heads=8, head_dim=128, context=32768,
           alpha_hh=0.10, alpha_rw=0.10, pyramid_depth=7, n_r=128, group_size=16)
# configs[4] (LWM-Text-7B, 32-head MHA, 256K context, batch 8 over 8 GPUs): one GPU's shard is one
# sequence; `--workload lwm-7b` measures that shard (decode + the 256K MHA prefill layer)
WORKLOADS = {
    "llama3-8b": dict(cfg=CFG, metric=METRIC,
                      desc="Llama-3-8B GQA decode, 32 layers, 32q/8kv heads, d=128, 32K context, "
                           "20% pyramid budget (10% HH depth-7 + 10% RW), n_r=128, group=16",
                      prefill=dict(name="Mistral-7B layer, 128K causal prefill (32q/8kv, d=128)", hq=32, hkv=8,
                                   L=131072)),
    "lwm-7b": dict(cfg=dict(CFG, batch=1, n_q_heads=32, n_kv_heads=32, context=262144),
                   metric="2-bit-KV decode attn tokens/s (LWM-Text-7B MHA, 256K ctx, 20% pyramid budget)",
                   desc="LWM-Text-7B MHA decode, 32 layers, 32 heads, d=128, 256K context, 20% pyramid budget "
                        "(10% HH depth-7 + 10% RW), n_r=128, group=16; one GPU's shard of configs[4]",
                   prefill=dict(name="LWM-Text-7B layer, 256K causal prefill (32 MHA heads, d=128)", hq=32, hkv=32,
                                L=262144)),
}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=40)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="mkv", choices=["mkv", "reference"])
    p.add_argument("--no-prefill", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--batch", type=int, default=None)
    p.add_argument("--workload", default="llama3-8b", choices=sorted(WORKLOADS))
    a = p.parse_args()
    if a.batch is None:
        a.batch = WORKLOADS[a.workload]["cfg"]["batch"]
    return a


def budgets(cfg):
    """Per-layer HH counts (pyramid, selection.cpp:61-83) and the RW count."""
    from paper_2411_18077_b200 import allocate_pyramid
    L = cfg["context"]
    x = int(math.floor(cfg["alpha_hh"] * L))
    rw = int(math.floor(cfg["alpha_rw"] * L))
    return allocate_pyramid(x, cfg["layers"], cfg["pyramid_depth"], True), rw


def budgets_host(cfg):
    import oracle
    L = cfg["context"]
    x = int(math.floor(cfg["alpha_hh"] * L))
    rw = int(math.floor(cfg["alpha_rw"] * L))
    return [int(v) for v in oracle.port().allocate_pyramid(x, cfg["layers"], cfg["pyramid_depth"], True)], rw


class ClockSampler:
    """SM clock and throttle reasons sampled DURING the timed region (NVML, 5 ms period;
    nvidia-smi as a fallback)."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4}

    def __init__(self, index=0):
        self.index, self.rows, self.stop = index, [], threading.Event()
        self.max_mhz = None

    def _poll(self):
        try:
            import pynvml as N
            N.nvmlInit()
            h = N.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
            while not self.stop.is_set():
                sm = N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)
                try:
                    rs = N.nvmlDeviceGetCurrentClocksEventReasons(h)
                except Exception:
                    rs = N.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                self.rows.append((sm, rs))
                time.sleep(0.005)
        except Exception:
            self.rows = []

    def __enter__(self):
        self.t = threading.Thread(target=self._poll, daemon=True)
        self.t.start()
        time.sleep(0.02)
        return self

    def __exit__(self, *a):
        self.stop.set()
        self.t.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"], "samples": 0}
        sm = [r[0] for r in self.rows]
        reasons = sorted({n for _, rs in self.rows for n, bit in self.REASONS.items() if rs & bit})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(self.rows)}


def load_traffic(kernel):
    """DRAM bytes per launch of `kernel` from the committed ncu capture (profiles/), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "r1_pages_traffic.json")) as f:
            t = json.load(f)
        return float(t["traffic_bytes_per_launch"]) if t.get("kernel") == kernel else None
    except Exception:
        return None


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), float(pk["bf16_tflops"]), float(pk.get("bf16_tflops_sustained", pk["bf16_tflops"])), "measured"
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback"


# ---------------------------------------------------------------------------
# the B200 arm
# ---------------------------------------------------------------------------
def run_mkv(args, rank, world):
    import torch
    import paper_2411_18077_b200 as mkv
    from paper_2411_18077_b200 import _capi
    import ctypes as C

    torch.cuda.set_device(rank % max(torch.cuda.device_count(), 1))
    dev = torch.device("cuda")
    _capi.check(_capi.lib().mkv_device_check(torch.cuda.current_device()), "device")
    cfg = dict(WORKLOADS[args.workload]["cfg"])
    cfg["batch"] = args.batch
    B, NL, Hq, Hkv, d, L = cfg["batch"], cfg["layers"], cfg["n_q_heads"], cfg["n_kv_heads"], cfg["head_dim"], cfg["context"]
    G = Hq // Hkv
    hh, rw = budgets(cfg)
    upl = B * Hkv                       # units per layer
    n_units = NL * upl                  # u = (layer * B + b) * Hkv + h
    steps_total = args.warmup + args.steps
    caps = [hh[l] + rw for l in range(NL) for _ in range(upl)]
    cache = mkv.KVCache(n_units, caps, max_decode_tokens=steps_total + cfg["n_r"], d=d, n_r=cfg["n_r"])
    stream = torch.cuda.current_stream()
    seed = SEED + 7919 * rank
    # ---- prefill the caches: synthetic fp16 K/V, synthetic A_cumul, select (K2) + pack (K3) ----
    t0 = time.time()
    for l in range(NL):
        u0 = l * upl
        k = mkv.synth_fp16((upl, L * d), seed, (2 << 48) | (u0 << 16), 1 << 16).view(upl, L, d)
        v = mkv.synth_fp16((upl, L * d), seed, (3 << 48) | (u0 << 16), 1 << 16).view(upl, L, d)
        a = mkv.synth_uniform((upl, L), seed, (7 << 48) | (u0 << 16), 1 << 16)
        cache.prefill(k, v, a, [hh[l]] * upl, rw, unit_begin=u0)
        del k, v, a
    cache.check()
    torch.cuda.synchronize()
    setup_s = time.time() - t0
    # ---- per-step inputs, resident in HBM before timing: stream (kind<<48)|(unit<<16)|(step+1) ----
    qs = torch.stack([mkv.synth_fp16((n_units, G * d), seed, (4 << 48) | (s + 1), 1 << 16)
                      for s in range(steps_total)]).view(steps_total, NL, upl, G, d)
    ks = torch.stack([mkv.synth_fp16((n_units, d), seed, (5 << 48) | (s + 1), 1 << 16)
                      for s in range(steps_total)]).view(steps_total, NL, upl, d)
    vs = torch.stack([mkv.synth_fp16((n_units, d), seed, (6 << 48) | (s + 1), 1 << 16)
                      for s in range(steps_total)]).view(steps_total, NL, upl, d)
    out = torch.empty((NL, upl, G, d), dtype=torch.float16, device=dev)
    scale = 1.0 / math.sqrt(d)
    L_ = _capi.lib()

    def step_args(s):
        arr = (_capi.DecodeArgs * NL)()
        for l in range(NL):
            arr[l] = _capi.DecodeArgs(l * upl, upl, G, qs[s, l].data_ptr(), ks[s, l].data_ptr(),
                                      vs[s, l].data_ptr(), out[l].data_ptr(), scale)
        return arr

    all_args = [step_args(s) for s in range(steps_total)]
    sp = int(stream.cuda_stream)

    def do_step(s):
        _capi.check(L_.mkv_decode_step_layers(cache.h, NL, all_args[s], sp), "decode")

    # pre-roll residual appends so that exactly one n_r flush lands inside the timed steps
    n_r = cfg["n_r"]
    preroll = max(0, n_r - args.warmup - args.steps // 2 - 1) if args.steps < n_r else 0
    for p in range(preroll):
        cache.append(ks[p % steps_total].view(n_units, d), vs[p % steps_total].view(n_units, d))
    pages_per_unit = [cache.unit_info(u)["n_pages"] for u in range(n_units)]
    base_pages = sum(pages_per_unit)

    # algorithmic bytes per step: pages (2-bit codes + fp16 params, K and V) +
    # fp16 residual K/V + q + out + the appended token.
    def step_bytes(step_index):
        t = preroll + step_index + 1
        r = t % n_r
        flushed = t // n_r
        pages = base_pages + flushed * n_units * (n_r // 16)
        return pages * 2048 + n_units * r * 4 * d + n_units * G * d * 2 * 2 + n_units * 2 * d * 2

    for s in range(args.warmup):
        do_step(s)
    torch.cuda.synchronize()
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(torch.cuda.current_device()) as clk:
        torch.cuda.synchronize()
        ev0.record(stream)
        for s in range(args.warmup, steps_total):
            do_step(s)
        ev1.record(stream)
        torch.cuda.synchronize()
    ms = dist_max(ev0.elapsed_time(ev1), world)
    ms_per_step = ms / args.steps
    bytes_timed = sum(step_bytes(s) for s in range(args.warmup, steps_total))
    tokens_per_s = world * B * args.steps / (ms / 1e3)
    res = dict(ms_per_step=ms_per_step, tokens_per_s=tokens_per_s,
               hbm_gbs=bytes_timed / (ms / 1e3) / 1e9 * world, clocks=clk.summary(), setup_s=setup_s,
               # per step: a page kernel + a finish kernel per layer; a flush step adds ONE append
               # launch for every layer and one plan-build launch (mkv_decode_step_layers)
               gpu_launches=args.steps * NL * 2 + 2 * sum(1 for s in range(args.warmup, steps_total)
                                                          if (preroll + s + 1) % n_r == 0),
               preroll=preroll,
               flushes_in_timed=sum(1 for s in range(args.warmup, steps_total) if (preroll + s + 1) % n_r == 0))
    # ---- dominant kernel alone (K4 page kernel), CUDA events on its stream ----
    reps = 20
    last = steps_total - 1
    attend_args = step_args(last)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        for l in range(NL):
            _capi.check(L_.mkv_decode_pages_only(cache.h, C.byref(attend_args[l]), sp), "pages")
    e1.record(stream)
    torch.cuda.synchronize()
    k_ms = e0.elapsed_time(e1) / (reps * NL)
    page_bytes_per_launch = (sum(cache.unit_info(u)["n_pages"] for u in range(n_units)) * 2048 +
                             n_units * G * d * 2 * 2) / NL
    res["kernel"] = dict(name="mkv::pages_kernel", avg_launch_ms=k_ms, bytes_per_launch=page_bytes_per_launch,
                         gbs=page_bytes_per_launch / (k_ms / 1e3) / 1e9)
    # ---- e2e through the C ABI with host buffers (pinned), copies inside the timed region.
    #      Serving-style pipelining: step s+2's inputs are copied in (H2D stream, 3 input
    #      buffers) and step s's outputs copied out (D2H stream, 2 output buffers) while the
    #      GPU computes; every dependency through CUDA events; the host reads step s-1's
    #      result (event sync) before issuing step s+1.  Wall clock over all steps. ----
    NIN, NOUT = 3, 2
    hq = qs[:, :, :, :, :].cpu().pin_memory()
    hk = ks.cpu().pin_memory()
    hv = vs.cpu().pin_memory()
    hout = [torch.empty((NL, upl, G, d), dtype=torch.float16).pin_memory() for _ in range(NOUT)]
    dq = [torch.empty((NL, upl, G, d), dtype=torch.float16, device=dev) for _ in range(NIN)]
    dk = [torch.empty((NL, upl, d), dtype=torch.float16, device=dev) for _ in range(NIN)]
    dv = [torch.empty((NL, upl, d), dtype=torch.float16, device=dev) for _ in range(NIN)]
    dout = [torch.empty((NL, upl, G, d), dtype=torch.float16, device=dev) for _ in range(NOUT)]
    e2e_args = {}
    for bi in range(NIN):
        for bo in range(NOUT):
            arr = (_capi.DecodeArgs * NL)()
            for l in range(NL):
                arr[l] = _capi.DecodeArgs(l * upl, upl, G, dq[bi][l].data_ptr(), dk[bi][l].data_ptr(),
                                          dv[bi][l].data_ptr(), dout[bo][l].data_ptr(), scale)
            e2e_args[bi, bo] = arr
    h2d, d2h = torch.cuda.Stream(), torch.cuda.Stream()
    e2e_steps = args.steps
    ev = lambda: [torch.cuda.Event() for _ in range(e2e_steps)]  # noqa: E731
    in_ready, computed, out_read = ev(), ev(), ev()

    def issue_h2d(s_):
        bi, src = s_ % NIN, (args.warmup + s_) % steps_total
        with torch.cuda.stream(h2d):
            if s_ >= NIN:
                h2d.wait_event(computed[s_ - NIN])  # the step that last read this input buffer
            dq[bi].copy_(hq[src], non_blocking=True)
            dk[bi].copy_(hk[src], non_blocking=True)
            dv[bi].copy_(hv[src], non_blocking=True)
            in_ready[s_].record(h2d)

    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for s in range(min(NIN - 1, e2e_steps)):
        issue_h2d(s)
    for s in range(e2e_steps):
        bi, bo = s % NIN, s % NOUT
        stream.wait_event(in_ready[s])
        if s >= NOUT:
            stream.wait_event(out_read[s - NOUT])  # that step's output has left this buffer
        _capi.check(L_.mkv_decode_step_layers(cache.h, NL, e2e_args[bi, bo], sp), "decode")
        computed[s].record(stream)
        if s + NIN - 1 < e2e_steps:
            issue_h2d(s + NIN - 1)
        with torch.cuda.stream(d2h):
            d2h.wait_event(computed[s])
            hout[bo].copy_(dout[bo], non_blocking=True)
            out_read[s].record(d2h)
        if s >= 1:
            out_read[s - 1].synchronize()  # the host reads step s-1's result
    out_read[e2e_steps - 1].synchronize()
    e2e_s = dist_max(time.perf_counter() - t0, world)
    res["e2e"] = dict(value=world * B * e2e_steps / e2e_s, unit=UNIT,
                      h2d_bytes_per_step=int(dq[0].numel() * 2 + dk[0].numel() * 2 + dv[0].numel() * 2),
                      d2h_bytes_per_step=int(dout[0].numel() * 2),
                      pipelining="H2D of step s+2 (3 input buffers) and D2H of step s-1 overlap step s "
                                 "(2 copy streams, events)")
    res["units"] = n_units
    res["pages"] = base_pages
    cache.close()
    return res


def run_prefill_bench(args):
    """K1 + K2 + K3 on the Mistral-7B-shaped 128K layer (configs[3]), or with --workload lwm-7b
    the LWM-Text-7B 256K MHA layer (configs[4])."""
    import torch
    import paper_2411_18077_b200 as mkv
    pw = WORKLOADS[args.workload]["prefill"]
    B, Hq, Hkv, d, L = 1, pw["hq"], pw["hkv"], 128, pw["L"]
    seed = SEED
    q = mkv.synth_fp16((B, Hq, L, d), seed, 1 << 48, 1 << 16)
    k = mkv.synth_fp16((B, Hkv, L, d), seed, 2 << 48, 1 << 16)
    v = mkv.synth_fp16((B, Hkv, L, d), seed, 3 << 48, 1 << 16)
    scale = 1.0 / math.sqrt(d)
    try:
        r = mkv.selective_flash_attn(q, k, v, scale, True)
    except mkv.MkvError as e:
        return {"unavailable": str(e)}
    torch.cuda.synchronize()
    reps = 3
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        r = mkv.selective_flash_attn(q, k, v, scale, True)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    P = L * (L + 1) / 2
    flops = Hq * 6 * d * P
    acs = float(r.a_cumul.double().sum().item())
    _, bf16_peak, _, _ = load_peaks()
    # exponentials: 2 per visible (query, key) pair (pass 1 and the A_cumul pass); the SFU
    # (MUFU.EX2) bound is 16 per clock per SM on B200 -- part of them run as FMA polynomials
    exps = 2.0 * Hq * P
    mufu_peak = 16.0 * torch.cuda.get_device_properties(0).multi_processor_count * 1.965e9
    out = {"workload": pw["name"], "ms": ms,
           "tflops": flops / (ms / 1e3) / 1e12, "frac_of_bf16_peak": flops / (ms / 1e3) / 1e12 / bf16_peak,
           "flop_count": "3 GEMM-eq = 6*d*L(L+1)/2 per q-head", "a_cumul_sum_over_G_lq": acs / (Hq * L),
           "exp_per_s": exps / (ms / 1e3), "exp_frac_of_mufu_peak": exps / (ms / 1e3) / mufu_peak,
           "exp_count": "2 per visible pair (pass 1 + A_cumul pass); MUFU peak 16/clk/SM at 1965 MHz, "
                        "a share of them evaluated on the FMA pipe (MKV_PREFILL_POLY)"}
    # K2 + K3 on the same layer at the 20% budget (10% HH + 10% RW): selection + gather/pack
    hh = rw = int(math.floor(0.10 * L))
    ac = r.a_cumul.view(Hkv, L)
    cache = mkv.KVCache(Hkv, hh + rw, 0)
    kk, vv = k.view(Hkv, L, d), v.view(Hkv, L, d)
    kept, nk = mkv.select_token_counts(ac, hh, rw)
    cache.prefill_kept(kk, vv, kept, nk)
    torch.cuda.synchronize()
    # K2 timed through the C ABI with prebuilt arguments (host overhead below the kernel's)
    import ctypes as C
    from paper_2411_18077_b200 import _capi
    hh_arr = (C.c_int32 * Hkv)(*([hh] * Hkv))
    sargs = _capi.SelectArgs(ac.data_ptr(), ac.stride(0), Hkv, L, hh_arr, rw, kept.data_ptr(), kept.stride(0), None)
    sp = int(torch.cuda.current_stream().cuda_stream)
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record()
    for _ in range(20):
        _capi.check(_capi.lib().mkv_select(C.byref(sargs), sp), "select")
    e[1].record()
    for _ in range(5):
        cache.prefill_kept(kk, vv, kept, nk)
    e[2].record()
    torch.cuda.synchronize()
    t2, t3 = e[0].elapsed_time(e[1]) / 20, e[1].elapsed_time(e[2]) / 5
    n_kept = hh + rw
    out["select_ms"] = t2
    out["select_gbs"] = Hkv * (4 * L + 4 * n_kept) / (t2 / 1e3) / 1e9
    out["pack_ms"] = t3
    out["pack_gbs"] = Hkv * n_kept * (4 * d + 4 + d) / (t3 / 1e3) / 1e9
    cache.close()
    # configs[3] budget sweep: total budget 10..50%, split evenly between HH and RW
    sweep = []
    for frac in (0.10, 0.20, 0.30, 0.40, 0.50):
        hh = rw = int(math.floor(frac / 2 * L))
        c2 = mkv.KVCache(Hkv, hh + rw, 0)
        kept, nk = mkv.select_token_counts(ac, hh, rw)
        c2.prefill_kept(kk, vv, kept, nk)
        torch.cuda.synchronize()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record()
        for _ in range(3):
            kept, nk = mkv.select_token_counts(ac, hh, rw)
        e[1].record()
        for _ in range(3):
            c2.prefill_kept(kk, vv, kept, nk)
        e[2].record()
        torch.cuda.synchronize()
        ts, tp = e[0].elapsed_time(e[1]) / 3, e[1].elapsed_time(e[2]) / 3
        sweep.append({"budget": frac, "kept_per_kv_head": hh + rw, "select_ms": round(ts, 4), "pack_ms": round(tp, 4),
                      "pack_gbs": round(Hkv * (hh + rw) * (4 * d + 4 + d) / (tp / 1e3) / 1e9, 1),
                      "cache_bytes": int(Hkv * (hh + rw) * d)})
        c2.close()
    out["budget_sweep"] = sweep
    return out


# ---------------------------------------------------------------------------
# reference CPU arm (oracle/_ref = the unmodified reference sources)
# ---------------------------------------------------------------------------
def cpu_reference_decode(steps, warmup, threads=None, sample_units_per_layer=4, cfg=CFG):
    """Time the reference decode on a bounded sample of cfg2 units; extrapolate to the
    whole step (linear in units: units are independent)."""
    import numpy as np
    import oracle
    R = oracle.ref()
    threads = threads or os.cpu_count() or 1
    hh, rw = budgets_host(cfg)
    B, NL, Hkv, G, d, L = cfg["batch"], cfg["layers"], cfg["n_kv_heads"], cfg["n_q_heads"] // cfg["n_kv_heads"], \
        cfg["head_dim"], cfg["context"]
    upl = B * Hkv
    sample = []
    for l in range(NL):
        for j in range(sample_units_per_layer):
            sample.append(l * upl + j)
    n = len(sample)
    hh_s = np.array([hh[u // upl] for u in sample], np.int64)
    ids = np.array(sample, np.uint64)
    import ctypes as C
    h = C.c_void_p()
    t0 = time.time()
    oracle._check(R.lib.mkr_decode_set_create(n, L, d, G, hh_s, rw, cfg["n_r"], cfg["group_size"], SEED, ids,
                                              threads, C.byref(h)), "decode_set_create")
    setup = time.time() - t0
    P = oracle.port()
    scale = 1.0 / math.sqrt(d)
    times = []
    out = np.zeros((n, G, d), np.float32)
    for s in range(warmup + steps):
        q = np.stack([P.synth_fp16(SEED, oracle.stream_id(oracle.KIND_QDEC, u, s + 1), G * d) for u in sample]).astype(np.float32)
        kk = np.stack([P.synth_fp16(SEED, oracle.stream_id(oracle.KIND_KDEC, u, s + 1), d) for u in sample]).astype(np.float32)
        vv = np.stack([P.synth_fp16(SEED, oracle.stream_id(oracle.KIND_VDEC, u, s + 1), d) for u in sample]).astype(np.float32)
        secs = C.c_double()
        oracle._check(R.lib.mkr_decode_set_step(h, np.ascontiguousarray(q), np.ascontiguousarray(kk),
                                                np.ascontiguousarray(vv), scale, out.reshape(-1), threads,
                                                C.byref(secs)), "decode_set_step")
        if s >= warmup:
            times.append(secs.value)
    R.lib.mkr_decode_set_destroy(h)
    t_sample = sum(times) / len(times)
    t_step = t_sample * (NL * upl) / n
    return {"value": B / t_step, "unit": UNIT, "cores": threads, "kind": "reference",
            "sample": f"{n} of {NL * upl} (layer, seq, kv-head) units ({sample_units_per_layer}/layer, every pyramid "
                      f"budget), L={L}, {steps} timed decode steps, {threads} threads; per-step time "
                      f"x{NL * upl / n:.0f} (units are independent)",
            "sample_step_s": t_sample, "setup_s": setup}


def dist_max(x: float, world: int) -> float:
    """Max of a per-rank scalar over all ranks (device timings are max-over-ranks)."""
    if world <= 1:
        return x
    import torch
    import torch.distributed as dist
    dev = "cpu" if dist.get_backend() == "gloo" else "cuda"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1 and args.impl == "mkv":
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")) % max(torch.cuda.device_count(), 1))
        # NCCL for the barrier / max-over-ranks reduction; MKV_DIST_BACKEND=gloo lets several
        # ranks share one GPU (the 1-GPU validation of the N > 1 path)
        dist.init_process_group(os.environ.get("MKV_DIST_BACKEND", "nccl"))
    hbm_peak, bf16_peak, bf16_sust, peak_kind = load_peaks()
    W = WORKLOADS[args.workload]
    metric = W["metric"]
    cfg_desc = {"workload": W["desc"],
                "batch_per_gpu": args.batch, "global_batch": args.batch * world, "context": W["cfg"]["context"],
                "parallelism": f"dp{world} (sequence-batch shards, no collective)",
                "l2": "inputs larger than L2 (GBs of 2-bit pages per step vs 126 MB L2)"}
    if args.impl == "reference":
        if rank != 0:
            return
        ref = cpu_reference_decode(args.steps, args.warmup, cfg=dict(W["cfg"], batch=args.batch))
        line = {"metric": metric, "value": ref["value"], "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * args.batch / ref["value"],
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
                "data": "synthetic (integer-exact N(0,1) fp16 K/V, uniform A_cumul)", "config": cfg_desc,
                "cpu_baseline": {k: ref[k] for k in ("value", "unit", "cores", "kind", "sample")},
                "e2e": {"value": ref["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return
    res = run_mkv(args, rank, world)
    prefill = None
    if not args.no_prefill and rank == 0:
        try:
            prefill = run_prefill_bench(args)
        except Exception as e:  # reported, never silently substituted
            prefill = {"error": repr(e)}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            import oracle
            if oracle.ref_available():
                cpu = cpu_reference_decode(steps=3, warmup=1, cfg=dict(W["cfg"], batch=args.batch))
            else:
                cpu = {"unavailable": "oracle/_ref not built"}
        except Exception as e:
            cpu = {"error": repr(e)}
    if rank != 0:
        return
    kern = res["kernel"]
    line = {
        "metric": metric, "value": res["tokens_per_s"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": res["ms_per_step"], "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "fp16 (2-bit codes, fp16 params, fp32 accumulate)",
        "data": "synthetic (integer-exact N(0,1) fp16 K/V/q, uniform A_cumul), random-init shapes",
        "config": cfg_desc,
        "hbm_gbs": res["hbm_gbs"],
        "roofline": {"bound": "hbm", "achieved": kern["gbs"], "peak": hbm_peak, "unit": "GB/s",
                     "frac": kern["gbs"] / hbm_peak,
                     "traffic": load_traffic(kern["name"]) if args.workload == "llama3-8b" else None,
                     "traffic_source": "profiles/r1_pages_traffic.json (ncu dram__bytes_read+write, mean of "
                                       "the 32 per-layer launches of one step)", "kernel": kern["name"],
                     "avg_launch_ms": kern["avg_launch_ms"], "bytes_per_launch": kern["bytes_per_launch"],
                     "peak_kind": peak_kind},
        "step_roofline_frac": res["hbm_gbs"] / (hbm_peak * world),
        "cpu_baseline": cpu, "e2e": res["e2e"], "gpu_launches": res["gpu_launches"], "clocks": res["clocks"],
        "prefill": prefill, "setup_s": res["setup_s"],
    }
    print(json.dumps(line))


if __name__ == "__main__":
    main()
