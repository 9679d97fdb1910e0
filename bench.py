#!/usr/bin/env python
"""bench.py -- MiniKV attention hot path on B200 (one JSON line on rank 0).

Headline workload: 2-bit-KV decode tokens/s for Llama-3-8B-shaped GQA attention (32 q / 8 kv
heads, d = 128, 32 layers, pyramid budget, 20% = 10% HH + 10% RW of a 32K context).

  * N = 1 (BASELINE.json configs[1]): batch 16 on one B200.
  * N > 1 (configs[2]): global batch 128 split by sequence over the N ranks
    (shard.plan: 64 / 32 / 16 sequences per GPU at N = 2 / 4 / 8; strong scaling, no
    collective on the attention path).  ``--workload lwm-7b`` is configs[4] (LWM-Text-7B
    MHA, 256K context, global batch 8 over the ranks; N = 1 runs one sequence's shard).

A "step" = one decode step through all 32 layers: per layer decode_append (+ the n_r flush)
and 2-bit attention over [pages ; residual] for every (seq, kv-head) unit (K4).  ``value``
is whole-job decode tokens/s with inputs resident in HBM, every layer's q known up front (the
reference arm's workload: independent units): one mkv_decode_step_layers call whose 32 layers
are laid out back to back, which the call runs as ONE page pass + ONE finish pass over all
(layer, seq, kv-head) units (MKV_LAYERS_SPLIT=1: one pass per layer, the A/B).  ``serving`` is
the same step as 32 mkv_decode_step calls with layer l+1's q = layer l's output (the
dependency a model has); ``e2e`` is ``value``'s form through the C ABI with pinned host buffers
copied in and out inside the timed region.

Also reported on rank 0 at N = 1: ``parity`` (the GPU decode outputs of the last timed step
vs the unmodified reference decode on the CPU sample units, same synthetic streams and the
same pre-roll), ``cpu_baseline`` (that reference decode timed on nproc threads and on one
thread), ``config0`` (BASELINE configs[0]: 8-head 4K prefill -> select -> pack -> 256
decode steps end to end on the GPU and in full on the CPU reference, with parity), and
``prefill`` (K1 at configs[3]'s Mistral-7B 128K layer, K2/K3 budget sweep, sampled-row /
column parity).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl mkv|reference]

``--gpus N`` with N > 1 outside torchrun re-launches itself under torch.distributed.run
(one rank per GPU, 127.0.0.1).  ``--impl reference`` times the reference CPU implementation
(oracle/_ref = the unmodified reference sources) on this host's cores, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import socket
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

UNIT = "tokens/s"
SEED = 2024
DECODE_TOL = 5e-3  # max |t_O - reference| (SURVEY 8(d) tolerances)
SPLIT = bool(os.environ.get("MKV_LAYERS_SPLIT"))  # A/B: one page + finish pass per layer

LLAMA = dict(layers=32, n_q_heads=32, n_kv_heads=8, head_dim=128, context=32768,
             alpha_hh=0.10, alpha_rw=0.10, pyramid_depth=7, n_r=128, group_size=16)
WORKLOADS = {
    "llama3-8b": dict(
        cfg=LLAMA, batch_n1=16, batch_multi=128,
        metric="2-bit-KV decode attn tokens/s (Llama-3-8B GQA, 32K ctx, 20% pyramid budget)",
        desc="Llama-3-8B GQA decode, 32 layers, 32q/8kv heads, d=128, 32K context, 20% pyramid budget "
             "(10% HH depth-7 + 10% RW), n_r=128, group=16",
        config_n1="configs[1]: batch 16 on 1xB200",
        config_multi="configs[2]: global batch 128 sharded by sequence over the GPUs",
        prefill=dict(name="Mistral-7B layer, 128K causal prefill (32q/8kv, d=128)", hq=32, hkv=8, L=131072)),
    "lwm-7b": dict(
        cfg=dict(LLAMA, n_q_heads=32, n_kv_heads=32, context=262144), batch_n1=1, batch_multi=8,
        metric="2-bit-KV decode attn tokens/s (LWM-Text-7B MHA, 256K ctx, 20% pyramid budget)",
        desc="LWM-Text-7B MHA decode, 32 layers, 32 heads, d=128, 256K context, 20% pyramid budget "
             "(10% HH depth-7 + 10% RW), n_r=128, group=16",
        config_n1="configs[4] shard: one sequence on 1xB200",
        config_multi="configs[4]: global batch 8 sharded by sequence over the GPUs",
        prefill=dict(name="LWM-Text-7B layer, 256K causal prefill (32 MHA heads, d=128)", hq=32, hkv=32, L=262144)),
}
# BASELINE configs[0]: single layer, 8 heads, d=128, 4K prefill + 256 decode steps, 20% budget
CFG0 = dict(heads=8, L=4096, d=128, alpha_hh=0.10, alpha_rw=0.10, steps=256, n_r=128, group_size=16)


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=40)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="mkv", choices=["mkv", "reference"])
    p.add_argument("--workload", default="llama3-8b", choices=sorted(WORKLOADS))
    p.add_argument("--batch", type=int, default=None, help="global batch (default: configs[1]/[2]/[4])")
    p.add_argument("--no-prefill", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-config0", action="store_true")
    p.add_argument("--no-serving", action="store_true")
    p.add_argument("--cpu-units-per-layer", type=int, default=4, help="reference decode sample per layer")
    return p.parse_args()


def global_batch(args, world):
    W = WORKLOADS[args.workload]
    if args.batch is not None:
        return args.batch
    return W["batch_n1"] if world == 1 else W["batch_multi"]


def budgets(cfg):
    """Per-layer HH counts (pyramid, selection.cpp:61-83; host arithmetic of the product) and RW."""
    from paper_2411_18077_b200 import allocate_pyramid
    L = cfg["context"]
    x = int(math.floor(cfg["alpha_hh"] * L))
    rw = int(math.floor(cfg["alpha_rw"] * L))
    return [int(h) for h in allocate_pyramid(x, cfg["layers"], cfg["pyramid_depth"], True)], rw


def budgets_host(cfg):
    import oracle
    L = cfg["context"]
    x = int(math.floor(cfg["alpha_hh"] * L))
    rw = int(math.floor(cfg["alpha_rw"] * L))
    return [int(v) for v in oracle.port().allocate_pyramid(x, cfg["layers"], cfg["pyramid_depth"], True)], rw


# ---------------------------------------------------------------------------
# clocks during the timed region: NVML polling thread, nvidia-smi as the fallback
# ---------------------------------------------------------------------------
class ClockSampler:
    """SM clock and throttle reasons sampled while the GPU phases run (NVML every 2 ms; when NVML
    is unavailable or yields nothing, the `nvidia-smi --query-gpu ... -lms 20` process that runs
    beside it)."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4}

    def __init__(self, index=0):
        self.index, self.rows, self.stop = index, [], threading.Event()
        self.max_mhz = None
        self.smi = None
        self.smi_file = None
        self.err = None

    def _poll(self):
        try:
            import pynvml as N
            N.nvmlInit()
            h = N.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
            get_reasons = getattr(N, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                N.nvmlDeviceGetCurrentClocksThrottleReasons
            while not self.stop.is_set():
                sm = N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)
                try:
                    rs = get_reasons(h)
                except Exception:
                    rs = 0
                self.rows.append((sm, rs))
                time.sleep(0.002)
        except Exception as e:  # fall back to nvidia-smi
            self.err = repr(e)

    def __enter__(self):
        try:
            self.smi_file = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
            self.smi = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=self.smi_file, stderr=subprocess.DEVNULL)
        except Exception:
            self.smi = None
        self.t = threading.Thread(target=self._poll, daemon=True)
        self.t.start()
        time.sleep(0.05)
        return self

    def __exit__(self, *a):
        time.sleep(0.03)
        self.stop.set()
        self.t.join(timeout=2)
        if self.smi is not None:
            self.smi.terminate()
            try:
                self.smi.wait(timeout=2)
            except Exception:
                self.smi.kill()

    def _smi_rows(self):
        rows, mx = [], None
        try:
            with open(self.smi_file.name) as f:
                for ln in f:
                    p = [x.strip() for x in ln.split(",")]
                    if len(p) < 6 or not p[0].isdigit():
                        continue
                    mx = int(p[1])
                    rs = 0
                    for bit, val in zip((0x8, 0x40, 0x20, 0x4), p[2:6]):
                        if val.lower() == "active":
                            rs |= bit
                    rows.append((int(p[0]), rs))
            os.unlink(self.smi_file.name)
        except Exception:
            pass
        return rows, mx

    def summary(self):
        rows, src = self.rows, "nvml"
        smi_rows, smi_max = self._smi_rows()
        if not rows and smi_rows:
            rows, src = smi_rows, "nvidia-smi"
            self.max_mhz = self.max_mhz or smi_max
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"], "samples": 0,
                    "source": None, "nvml_error": self.err}
        sm = [r[0] for r in rows]
        reasons = sorted({n for _, rs in rows for n, bit in self.REASONS.items() if rs & bit})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(rows), "source": src, "nvidia_smi_samples": len(smi_rows)}


def load_traffic(kernel, launch_units):
    """DRAM bytes per launch of `kernel` over `launch_units` units from the newest committed ncu
    capture of that launch shape (profiles/), or None."""
    for name in ("r2_pages_traffic_all_layers.json", "r2_pages_traffic.json", "r1_pages_traffic.json"):
        try:
            with open(os.path.join(ROOT, "profiles", name)) as f:
                t = json.load(f)
            if t.get("kernel") == kernel and t.get("launch_units", 128) == launch_units:
                return float(t["traffic_bytes_per_launch"]), f"profiles/{name}"
        except Exception:
            continue
    return None, None


def host_cpu():
    """The GPU host's CPU as the CPU baselines ran on it (record nproc and lscpu)."""
    info = {"nproc": os.cpu_count()}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            k, _, v = line.partition(":")
            if k.strip() in ("Model name", "Socket(s)", "Core(s) per socket", "Thread(s) per core", "CPU max MHz"):
                info[k.strip()] = v.strip()
    except Exception:
        try:
            with open("/proc/cpuinfo") as f:
                info["Model name"] = next(l.split(":", 1)[1].strip() for l in f if l.startswith("model name"))
        except Exception:
            pass
    return info


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), float(pk["bf16_tflops"]), float(pk.get("bf16_tflops_sustained", pk["bf16_tflops"])), "measured"
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback"


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


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


# ---------------------------------------------------------------------------
# the B200 arm: decode
# ---------------------------------------------------------------------------
def rank_units(args, rank, world):
    """This rank's shard (shard.plan) as per-layer contiguous global unit ranges.  Global unit id
    u = (layer * B + b) * Hkv + h: the synthetic streams depend only on it, so every N sees the
    same data for the same unit."""
    from paper_2411_18077_b200 import shard
    cfg = WORKLOADS[args.workload]["cfg"]
    B, Hkv = global_batch(args, world), cfg["n_kv_heads"]
    sh = shard.plan(B, Hkv, world, rank)
    b0, nb = sh.seqs[0], len(sh.seqs)
    h0, nh = sh.kv_heads[0], len(sh.kv_heads)
    # contiguous: batch-major shards own whole sequences (all heads); head-split shards own one
    # sequence's head range
    assert list(sh.seqs) == list(range(b0, b0 + nb)) and list(sh.kv_heads) == list(range(h0, h0 + nh))
    assert nh == Hkv or nb == 1
    firsts = [(l * B + b0) * Hkv + h0 for l in range(cfg["layers"])]
    return sh, firsts, nb * nh


def run_mkv(args, rank, world):
    import ctypes as C

    import torch

    import paper_2411_18077_b200 as mkv
    from paper_2411_18077_b200 import _capi

    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")) % max(torch.cuda.device_count(), 1))
    dev = torch.device("cuda")
    _capi.check(_capi.lib().mkv_device_check(torch.cuda.current_device()), "device")
    cfg = WORKLOADS[args.workload]["cfg"]
    NL, Hq, Hkv, d, L, n_r = cfg["layers"], cfg["n_q_heads"], cfg["n_kv_heads"], cfg["head_dim"], cfg["context"], cfg["n_r"]
    G = Hq // Hkv
    hh, rw = budgets(cfg)
    sh, firsts, upl = rank_units(args, rank, world)
    B_local = len(sh.seqs)
    n_units = NL * upl                       # local unit i = l * upl + j  <->  global firsts[l] + j
    steps_total = args.warmup + args.steps
    caps = [hh[l] + rw for l in range(NL) for _ in range(upl)]
    # room for: pre-roll + timed + serving + e2e windows (+ one n_r block of slack)
    max_dec = n_r + 4 * steps_total + n_r
    cache = mkv.KVCache(n_units, caps, max_decode_tokens=max_dec, d=d, n_r=n_r)
    stream = torch.cuda.current_stream()
    seed = SEED
    # ---- prefill the caches: synthetic fp16 K/V, synthetic A_cumul, select (K2) + pack (K3) ----
    t0 = time.time()
    for l in range(NL):
        u0 = firsts[l]
        k = mkv.synth_fp16((upl, L * d), seed, (2 << 48) | (u0 << 16), 1 << 16).view(upl, L, d)
        v = mkv.synth_fp16((upl, L * d), seed, (3 << 48) | (u0 << 16), 1 << 16).view(upl, L, d)
        a = mkv.synth_uniform((upl, L), seed, (7 << 48) | (u0 << 16), 1 << 16)
        cache.prefill(k, v, a, [hh[l]] * upl, rw, unit_begin=l * upl)
        del k, v, a
    cache.check()
    torch.cuda.synchronize()
    setup_s = time.time() - t0

    # ---- per-step inputs, resident in HBM before timing: stream (kind<<48)|(u_global<<16)|(step+1) ----
    def step_inputs(s):
        q = torch.empty((NL, upl, G * d), dtype=torch.float16, device=dev)
        kk = torch.empty((NL, upl, d), dtype=torch.float16, device=dev)
        vv = torch.empty((NL, upl, d), dtype=torch.float16, device=dev)
        for l in range(NL):
            base = firsts[l] << 16
            q[l] = mkv.synth_fp16((upl, G * d), seed, (4 << 48) | base | (s + 1), 1 << 16)
            kk[l] = mkv.synth_fp16((upl, d), seed, (5 << 48) | base | (s + 1), 1 << 16)
            vv[l] = mkv.synth_fp16((upl, d), seed, (6 << 48) | base | (s + 1), 1 << 16)
        return q.view(NL, upl, G, d), kk, vv
    ins = [step_inputs(s) for s in range(steps_total)]
    qs = torch.stack([x[0] for x in ins])
    ks = torch.stack([x[1] for x in ins])
    vs = torch.stack([x[2] for x in ins])
    del ins
    out = torch.empty((NL, upl, G, d), dtype=torch.float16, device=dev)
    scale = 1.0 / math.sqrt(d)
    L_ = _capi.lib()
    sp = int(stream.cuda_stream)

    def layer_args(s, l, q_ptr=None, out_t=None):
        o = out if out_t is None else out_t
        return _capi.DecodeArgs(l * upl, upl, G, q_ptr if q_ptr is not None else qs[s, l].data_ptr(),
                                ks[s, l].data_ptr(), vs[s, l].data_ptr(), o[l].data_ptr(), scale)

    def step_args(s):
        arr = (_capi.DecodeArgs * NL)()
        for l in range(NL):
            arr[l] = layer_args(s, l)
        return arr

    all_args = [step_args(s) for s in range(steps_total)]

    def do_step(s):
        # q / k / v / out of the 32 layers are back to back ([NL, upl, ...]): the call coalesces
        # them into one page pass + one finish pass over all n_units (MKV_LAYERS_SPLIT=1: one per layer)
        _capi.check(L_.mkv_decode_step_layers(cache.h, NL, all_args[s], sp), "decode")

    # pre-roll residual appends so that exactly one n_r flush lands inside the timed steps (the
    # token of pre-roll append p is the decode token of step p % steps_total; the CPU parity run
    # replays the same appends)
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
    barrier(world)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clk = ClockSampler(torch.cuda.current_device())
    clk.__enter__()
    torch.cuda.synchronize()
    from paper_2411_18077_b200 import _capi
    launches0 = int(_capi.lib().mkv_debug_launch_count())
    ev0.record(stream)
    for s in range(args.warmup, steps_total):
        do_step(s)
    ev1.record(stream)
    torch.cuda.synchronize()
    launches_timed = int(_capi.lib().mkv_debug_launch_count()) - launches0
    ms = dist_max(ev0.elapsed_time(ev1), world)
    # outputs of the last timed step, for the parity check against the reference
    last_out = out.float().cpu()
    ms_per_step = ms / args.steps
    bytes_timed = sum(step_bytes(s) for s in range(args.warmup, steps_total))
    B_global = global_batch(args, world)
    tokens_per_s = B_global * args.steps / (ms / 1e3)
    flushes = sum(1 for s in range(args.warmup, steps_total) if (preroll + s + 1) % n_r == 0)
    res = dict(ms_per_step=ms_per_step, tokens_per_s=tokens_per_s,
               hbm_gbs=dist_max(bytes_timed, 1) / (ms / 1e3) / 1e9,
               setup_s=setup_s, preroll=preroll, flushes_in_timed=flushes,
               # counted by the library (mkv_debug_launch_count) over the timed steps: per step a
               # page kernel + residual + merge kernel (calls with more units than SMs) or + one
               # finish kernel; a flush step adds the append launch
               gpu_launches=launches_timed,
               B_local=B_local, upl=upl, n_units=n_units, pages=base_pages)
    # bytes of every rank (whole-job GB/s)
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([float(bytes_timed)], dtype=torch.float64,
                         device="cpu" if dist.get_backend() == "gloo" else "cuda")
        dist.all_reduce(t)
        res["hbm_gbs"] = float(t.item()) / (ms / 1e3) / 1e9

    # ---- serving-realistic: one mkv_decode_step per layer, layer l+1's q = layer l's output ----
    if not args.no_serving:
        outs = torch.empty((2, NL, upl, G, d), dtype=torch.float16, device=dev)
        s_steps = args.steps

        def serve_step(s, buf):
            src = args.warmup + (s % args.steps)
            o = outs[buf]
            for l in range(NL):
                qp = qs[src, 0].data_ptr() if l == 0 else o[l - 1].data_ptr()
                a = layer_args(src, l, q_ptr=qp, out_t=o)
                _capi.check(L_.mkv_decode_step(cache.h, C.byref(a), sp), "decode")
        for s in range(min(3, s_steps)):
            serve_step(s, s & 1)
        torch.cuda.synchronize()
        barrier(world)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        th0 = time.perf_counter()
        for s in range(s_steps):
            serve_step(s, s & 1)
        host_ms = (time.perf_counter() - th0) * 1e3  # the host's issue time (runs ahead of the GPU)
        e1.record(stream)
        torch.cuda.synchronize()
        sms = dist_max(e0.elapsed_time(e1), world)
        res["serving"] = dict(
            ms_per_step=sms / s_steps, tokens_per_s=B_global * s_steps / (sms / 1e3),
            step_roofline_frac_approx=(bytes_timed / args.steps) / (sms / s_steps / 1e3) / 1e9 / load_peaks()[0],
            how="32 mkv_decode_step calls per step; layer l+1's q is layer l's output (device buffer, "
                "no host round trip): each page kernel waits for the previous layer's merge",
            host_issue_ms_per_step=host_ms / s_steps, steps=s_steps)

    # ---- dominant kernel alone (K4 page kernel, as the timed steps launch it: one launch over
    #      all n_units, or one per layer under MKV_LAYERS_SPLIT), CUDA events on its stream ----
    reps = 20
    s_last = steps_total - 1
    attend_args = step_args(s_last) if SPLIT else [
        _capi.DecodeArgs(0, n_units, G, qs[s_last].data_ptr(), None, None, out.data_ptr(), scale)]
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        for a_ in attend_args:
            _capi.check(L_.mkv_decode_pages_only(cache.h, C.byref(a_), sp), "pages")
    e1.record(stream)
    torch.cuda.synchronize()
    k_ms = e0.elapsed_time(e1) / (reps * len(attend_args))
    page_bytes_per_launch = (sum(cache.unit_info(u)["n_pages"] for u in range(n_units)) * 2048 +
                             n_units * G * d * 2 * 2) / len(attend_args)
    res["kernel"] = dict(name="mkv::pages_kernel", avg_launch_ms=k_ms, bytes_per_launch=page_bytes_per_launch,
                         launch_units=n_units // len(attend_args),
                         gbs=page_bytes_per_launch / (k_ms / 1e3) / 1e9)

    # ---- e2e through the C ABI with host buffers (pinned), copies inside the timed region.
    #      Serving-style pipelining: step s+2's inputs are copied in (H2D stream, 3 input
    #      buffers) and step s's outputs copied out (D2H stream, 2 output buffers) while the
    #      GPU computes; every dependency through CUDA events; the host reads step s-1's
    #      result (event sync) before issuing step s+1.  Wall clock over all steps. ----
    NIN, NOUT = 3, 2
    hq = qs.cpu().pin_memory()
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
    barrier(world)
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
    clk.__exit__()
    res["clocks"] = clk.summary()
    res["clocks"]["window"] = "timed decode steps + serving + page-kernel roofline + e2e"
    res["e2e"] = dict(value=B_global * e2e_steps / e2e_s, unit=UNIT,
                      h2d_bytes_per_step=int(dq[0].numel() * 2 + dk[0].numel() * 2 + dv[0].numel() * 2),
                      d2h_bytes_per_step=int(dout[0].numel() * 2),
                      pipelining="H2D of step s+2 (3 input buffers) and D2H of step s-1 overlap step s "
                                 "(2 copy streams, events)")
    res["last_out"] = last_out
    res["steps_total"] = steps_total
    res["firsts"] = firsts
    cache.close()
    return res


# ---------------------------------------------------------------------------
# the reference's decode on a sample of units: timing (cpu_baseline / reference arm) and parity
# ---------------------------------------------------------------------------
def reference_decode(cfg, B, steps_total, preroll, timed_from, threads, units_per_layer, compare=None,
                     one_thread_steps=0):
    """The unmodified reference decode (oracle/_ref: decode_append + stored_keys/values +
    decode_attention per q-head, cache_engine.cpp / attention.cpp) over `units_per_layer` units of
    every layer (b = 0, kv-heads 0..; every pyramid budget), on `threads` host threads.
    Replays the GPU arm's pre-roll appends and decode steps 0..steps_total-1 with the same
    synthetic streams; steps >= timed_from are timed.  compare = (gpu_out [NL, upl, G, d] of the
    last step, upl) -> max |gpu - reference| over the sample."""
    import ctypes as C

    import numpy as np

    import oracle
    R = oracle.ref()
    P = oracle.port()
    hh, rw = budgets_host(cfg)
    NL, Hkv, G, d, L = cfg["layers"], cfg["n_kv_heads"], cfg["n_q_heads"] // cfg["n_kv_heads"], cfg["head_dim"], \
        cfg["context"]
    upl_g = B * Hkv
    sample = [l * upl_g + j for l in range(NL) for j in range(min(units_per_layer, upl_g))]
    n = len(sample)
    hh_s = np.array([hh[u // upl_g] for u in sample], np.int64)
    ids = np.array(sample, np.uint64)
    h = C.c_void_p()
    t0 = time.time()
    oracle._check(R.lib.mkr_decode_set_create(n, L, d, G, hh_s, rw, cfg["n_r"], cfg["group_size"], SEED, ids,
                                              threads, C.byref(h)), "decode_set_create")
    setup = time.time() - t0
    scale = 1.0 / math.sqrt(d)

    def tok(kind, s, width):
        return np.ascontiguousarray(np.stack([P.synth_fp16(SEED, oracle.stream_id(kind, u, s + 1), width)
                                              for u in sample]).astype(np.float32))
    for p in range(preroll):
        s = p % steps_total
        oracle._check(R.lib.mkr_decode_set_append(h, tok(oracle.KIND_KDEC, s, d), tok(oracle.KIND_VDEC, s, d),
                                                  threads), "decode_set_append")
    times = []
    out = np.zeros((n, G, d), np.float32)
    for s in range(steps_total):
        q, kk, vv = tok(oracle.KIND_QDEC, s, G * d), tok(oracle.KIND_KDEC, s, d), tok(oracle.KIND_VDEC, s, d)
        secs = C.c_double()
        oracle._check(R.lib.mkr_decode_set_step(h, q, kk, vv, scale, out.reshape(-1), threads, C.byref(secs)),
                      "decode_set_step")
        if s >= timed_from:
            times.append(secs.value)
    res = {"units": n, "units_total": NL * upl_g, "setup_s": setup, "step_times": times,
           "sample_step_s": sum(times) / max(len(times), 1), "threads": threads}
    if compare is not None:
        gpu, upl = compare
        worst = 0.0
        for i, u in enumerate(sample):
            l, j = divmod(u, upl_g)
            worst = max(worst, float(np.max(np.abs(gpu[l, j].numpy() - out[i]))))
        res["max_abs"] = worst
    if one_thread_steps:
        t1 = []
        for s in range(one_thread_steps):
            src = s % steps_total
            q, kk, vv = tok(oracle.KIND_QDEC, src, G * d), tok(oracle.KIND_KDEC, src, d), tok(oracle.KIND_VDEC, src, d)
            secs = C.c_double()
            oracle._check(R.lib.mkr_decode_set_step(h, q, kk, vv, scale, out.reshape(-1), 1, C.byref(secs)),
                          "decode_set_step")
            t1.append(secs.value)
        res["one_thread_step_s"] = sum(t1) / len(t1)
    R.lib.mkr_decode_set_destroy(h)
    return res


# ---------------------------------------------------------------------------
# configs[0]: the single-layer chain the reference CLI runs, end to end on both arms
# ---------------------------------------------------------------------------
def config0_gpu():
    """K1 prefill attention -> K2 select -> K3 pack -> 256 K4 decode steps, 8 heads x 4K, on
    cuda:0, device-timed (inputs resident) and end to end from pinned host buffers."""
    import torch

    import paper_2411_18077_b200 as mkv
    c = CFG0
    H, L, d, steps, n_r = c["heads"], c["L"], c["d"], c["steps"], c["n_r"]
    hh = int(math.floor(c["alpha_hh"] * L))
    rw = int(math.floor(c["alpha_rw"] * L))
    scale = 1.0 / math.sqrt(d)
    q = mkv.synth_fp16((H, L * d), SEED, 1 << 48, 1 << 16).view(1, H, L, d)
    k = mkv.synth_fp16((H, L * d), SEED, 2 << 48, 1 << 16).view(1, H, L, d)
    v = mkv.synth_fp16((H, L * d), SEED, 3 << 48, 1 << 16).view(1, H, L, d)
    qd = torch.stack([mkv.synth_fp16((H, d), SEED, (4 << 48) | (s + 1), 1 << 16) for s in range(steps)]).view(steps, H, 1, d)
    kd = torch.stack([mkv.synth_fp16((H, d), SEED, (5 << 48) | (s + 1), 1 << 16) for s in range(steps)])
    vd = torch.stack([mkv.synth_fp16((H, d), SEED, (6 << 48) | (s + 1), 1 << 16) for s in range(steps)])
    outs = torch.empty((steps, H, 1, d), dtype=torch.float16, device="cuda")

    def new_cache():  # the device pool: allocated once per chain, OUTSIDE the timed regions (a
        # serving engine holds it across requests); its cost is reported as make_cache_ms
        return mkv.KVCache(H, hh + rw, max_decode_tokens=steps + n_r, n_r=n_r)

    def chain(cache, qq, kk, vv, qdd, kdd, vdd, ev=None):
        r = mkv.selective_flash_attn(qq, kk, vv, scale, True)
        if ev:
            ev[1].record()
        cache.prefill(kk[0], vv[0], r.a_cumul[0], hh, rw)
        if ev:
            ev[2].record()
        cache.decode_steps(qdd, kdd, vdd, scale, out=outs)  # the 256 steps in one FFI crossing
        return r

    # warm-up: module load, kernel attributes, and at least ~0.3 s of GPU work so the clocks are
    # back up after the CPU phases that precede this leg (a short chain is launch-bound)
    t_w = time.perf_counter()
    n_w = 0
    while n_w < 2 or time.perf_counter() - t_w < 0.3:
        cache = new_cache()
        r = chain(cache, q, k, v, qd, kd, vd)
        torch.cuda.synchronize()
        cache.close()
        n_w += 1
    times, allocs = [], []
    for _ in range(9):  # median of 9 timed chains
        t0 = time.perf_counter()
        cache = new_cache()
        torch.cuda.synchronize()
        allocs.append((time.perf_counter() - t0) * 1e3)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        ev[0].record()
        r = chain(cache, q, k, v, qd, kd, vd, ev)
        ev[3].record()
        torch.cuda.synchronize()
        cache.close()
        times.append((ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2]), ev[2].elapsed_time(ev[3])))
    times.sort(key=lambda x: sum(x))
    t_attn, t_pack, t_dec = times[len(times) // 2]
    kept, nk = mkv.select_token_counts(r.a_cumul[0], hh, rw)
    gpu_out = outs.float().cpu().numpy()
    gpu_xo = r.output.float().cpu().numpy()[0]
    gpu_kept = kept.cpu().numpy()
    # end to end: Q/K/V and the decode tokens copied from pinned host memory inside the timed
    # region, every step's output read back by the host
    hq, hk, hv = q.cpu().pin_memory(), k.cpu().pin_memory(), v.cpu().pin_memory()
    hqd, hkd, hvd = qd.cpu().pin_memory(), kd.cpu().pin_memory(), vd.cpu().pin_memory()
    hout = torch.empty_like(outs, device="cpu").pin_memory()
    e2es = []
    for _ in range(5):  # median of 5
        cache = new_cache()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        dq, dk, dv = hq.cuda(non_blocking=True), hk.cuda(non_blocking=True), hv.cuda(non_blocking=True)
        dqd, dkd, dvd = hqd.cuda(non_blocking=True), hkd.cuda(non_blocking=True), hvd.cuda(non_blocking=True)
        chain(cache, dq, dk, dv, dqd, dkd, dvd)
        hout.copy_(outs, non_blocking=True)
        torch.cuda.synchronize()
        e2es.append((time.perf_counter() - t0) * 1e3)
        cache.close()
    e2e_ms = sorted(e2es)[len(e2es) // 2]
    # the same 256 decode steps as one mkv_decode_step call per step (the form a model's token
    # loop drives, each step's q known only when it is issued), device-timed after an untimed
    # prefill; outputs checked against the token-stream kernel's
    per_step = []
    outs1 = torch.empty_like(outs)
    for _ in range(5):  # median of 5
        cache = new_cache()
        r1 = mkv.selective_flash_attn(q, k, v, scale, True)
        cache.prefill(k[0], v[0], r1.a_cumul[0], hh, rw)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record()
        for s in range(steps):
            cache.decode_step(qd[s].view(H, 1, d), kd[s], vd[s], scale, out=outs1[s].view(H, 1, d))
        ev[1].record()
        torch.cuda.synchronize()
        per_step.append(ev[0].elapsed_time(ev[1]))
        cache.close()
    per_step_ms = sorted(per_step)[len(per_step) // 2]
    per_step_dev = float((outs1.float() - outs.float()).abs().max().item())
    total_ms = t_attn + t_pack + t_dec
    P = L * (L + 1) / 2
    return {
        "workload": "configs[0]: 1 layer, 8 heads (MHA), d=128, 4K causal prefill (K1) -> 20% budget select (K2, "
                    "409 HH + 409 RW) -> 2-bit pack (K3) -> 256 decode steps (K4, 2 flushes)",
        "gpu_ms": {"prefill_attn": t_attn, "select_pack": t_pack, "decode_256": t_dec, "total": total_ms,
                   "e2e_total_from_host": e2e_ms, "make_cache_outside_timing": sorted(allocs)[len(allocs) // 2],
                   "decode_256_per_step_calls": per_step_ms},
        "per_step_calls": {"how": "256 mkv_decode_step calls (one per step, q of step s issued with step s), "
                                  "device time after an untimed prefill; the headline chain's decode_256 runs the "
                                  "same steps as one mkv_decode_steps call over the prepared token stream, as the "
                                  "reference CLI's loop over its stream does",
                           "max_abs_vs_decode_steps": per_step_dev},
        "how": "make_cache (the device pool allocation) before the timed region; K1 -> K2+K3 -> "
               "256 decode steps through KVCache.decode_steps (mkv_decode_steps: one FFI crossing); "
               "e2e copies Q/K/V and the decode tokens from pinned host buffers and reads every output back",
        "gpu_prefill_tflops": H * 6 * d * P / (t_attn / 1e3) / 1e12,
        "gpu_decode_tokens_per_s": steps / (t_dec / 1e3),
        "h2d_bytes": int((q.numel() + k.numel() + v.numel() + qd.numel() + kd.numel() + vd.numel()) * 2),
        "d2h_bytes": int(outs.numel() * 2),
        "_out": gpu_out[:, :, 0, :], "_xo": gpu_xo, "_kept": gpu_kept, "_nk": nk, "_hh": hh, "_rw": rw,
    }


def config0_cpu(threads_list, hh, rw):
    """The reference chain (selective_flash_attn -> prefill -> decode_step x 256, ref_capi.cpp
    mkr_pipeline_run) for the 8 heads of configs[0], timed in full at each thread count."""
    import oracle
    R = oracle.ref()
    c = CFG0
    res = {}
    first = None
    for th in threads_list:
        r = R.pipeline_run(c["heads"], 1, c["L"], c["d"], hh, rw, c["steps"], SEED, th, c["n_r"], c["group_size"],
                           want_xo=first is None)
        res[th] = {"wall_s": r["wall_s"], "attn_thread_s": r["attn_thread_s"],
                   "prefill_thread_s": r["prefill_thread_s"], "decode_thread_s": r["decode_thread_s"]}
        if first is None:
            first = r
    return res, first


def config0(threads):
    import numpy as np
    g = config0_gpu()
    hh, rw = g.pop("_hh"), g.pop("_rw")
    ths = sorted({1, threads})
    cpu, ref = config0_cpu(ths, hh, rw)
    gk, gnk = g.pop("_kept"), g.pop("_nk")
    same_sel = [bool(np.array_equal(gk[h, :gnk[h]].astype(np.int64), ref["kept"][h, :ref["n_kept"][h]]))
                for h in range(CFG0["heads"])]
    gout, gxo = g.pop("_out"), g.pop("_xo")
    dec_dev = [float(np.max(np.abs(gout[:, h] - ref["out"][:, h]))) for h in range(CFG0["heads"]) if same_sel[h]]
    xo_dev = float(np.max(np.abs(gxo - ref["x_o"])))
    # the reference's prefill attention rate (3 GEMM-equivalents, 6 d P per head, P = L(L+1)/2),
    # measured on the 8 x 4K heads: thread-seconds of selective_flash_attn on one thread
    P0 = CFG0["L"] * (CFG0["L"] + 1) / 2
    for t_, v_ in cpu.items():
        v_["attn_gflops_per_thread"] = CFG0["heads"] * 6 * CFG0["d"] * P0 / v_["attn_thread_s"] / 1e9
    g["cpu_reference"] = {str(t): v for t, v in cpu.items()}
    g["cpu_reference"]["kind"] = "reference (oracle/_ref, unmodified sources; one thread per head)"
    g["speedup_vs_cpu_nproc"] = cpu[threads]["wall_s"] * 1e3 / g["gpu_ms"]["e2e_total_from_host"]
    g["speedup_vs_cpu_1thread"] = cpu[1]["wall_s"] * 1e3 / g["gpu_ms"]["e2e_total_from_host"]
    g["parity"] = {"x_o_max_abs": xo_dev, "x_o_tol": 5e-3,
                   "kept_identical_heads": int(sum(same_sel)), "heads": CFG0["heads"],
                   "decode_max_abs_all_256_steps": max(dec_dev) if dec_dev else None, "decode_tol": DECODE_TOL,
                   "note": "selection compares the device A_cumul's top-k with the reference's fp32 A_cumul "
                           "(different summation order: a near-tie at the budget boundary can swap one index; "
                           "decode parity is reported for the heads whose kept sets agree)",
                   "ok": bool(xo_dev <= 5e-3 and (not dec_dev or max(dec_dev) <= DECODE_TOL))}
    return g


# ---------------------------------------------------------------------------
# prefill (configs[3]): K1 + K2 + K3, sampled-row / column parity
# ---------------------------------------------------------------------------
def prefill_parity(q, k, v, r, Hq, Hkv, L, d, scale, rows, cols):
    """Sampled rows (X_O, LSE) against the reference's single-query attention over the row's
    visible keys (oracle port decode_attention, attention.cpp:119-143 = row i of
    selective_flash_attn), and sampled A_cumul columns recomputed on the host in fp64 from Q, k_j
    and the device LSE (pass 2 is a function of the LSE, attention.cpp:101-115)."""
    import numpy as np

    import oracle
    P = oracle.port()
    G = Hq // Hkv
    lse = r.lse[0].float().cpu().numpy()            # [Hq, L]
    xo_w, lse_w = 0.0, 0.0
    for h in range(0, Hq, max(1, Hq // 4)):
        kh = k[0, h // G].float().cpu().numpy()
        vh = v[0, h // G].float().cpu().numpy()
        for i in rows:
            qi = q[0, h, i].float().cpu().numpy()
            o, _ = P.decode_attention(qi, kh[:i + 1], vh[:i + 1], scale)
            xo_w = max(xo_w, float(np.max(np.abs(r.output[0, h, i].float().cpu().numpy() - o))))
            s = (kh[:i + 1].astype(np.float64) @ qi.astype(np.float64)) * scale
            m = s.max()
            lse_w = max(lse_w, abs(float(lse[h, i]) - (m + math.log(np.exp(s - m).sum()))))
    ac = r.a_cumul[0].cpu().numpy()                 # [Hkv, L]
    col_w, col_rel = 0.0, 0.0
    for hk in range(0, Hkv, max(1, Hkv // 2)):
        kc = k[0, hk][cols].float().cpu().numpy().astype(np.float64)    # [ncol, d]
        exp = np.zeros(len(cols))
        for g in range(G):
            h = hk * G + g
            qh = q[0, h].float().cpu().numpy().astype(np.float64)         # [L, d]
            s = qh @ kc.T * scale                                          # [L, ncol]
            e = np.exp(s - lse[h].astype(np.float64)[:, None])
            for ci, j in enumerate(cols):
                exp[ci] += e[j:, ci].sum()                                 # causal: rows i >= j see j
        got = ac[hk, cols]
        col_w = max(col_w, float(np.max(np.abs(got - exp) - 2e-3 * np.abs(exp))))
        col_rel = max(col_rel, float(np.max(np.abs(got - exp) / np.maximum(np.abs(exp), 1e-30))))
    return {"rows": list(rows), "cols": list(cols), "x_o_max_abs": xo_w, "x_o_tol": 5e-3, "lse_max_abs": lse_w,
            "lse_tol": 1e-3, "a_cumul_excess_over_rel_tol": col_w, "a_cumul_max_rel": col_rel,
            "a_cumul_tol": "|d| <= 1e-3 + 2e-3|ref|",
            "ok": bool(xo_w <= 5e-3 and lse_w <= 1e-3 and col_w <= 1e-3)}


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
    reps = []
    for _ in range(5):  # median of 5 launches (each timed with CUDA events)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r = mkv.selective_flash_attn(q, k, v, scale, True)
        e1.record()
        torch.cuda.synchronize()
        reps.append(e0.elapsed_time(e1))
    ms = sorted(reps)[len(reps) // 2]
    P = L * (L + 1) / 2
    flops = Hq * 6 * d * P
    acs = float(r.a_cumul.double().sum().item())
    _, bf16_peak, bf16_sustained, _ = load_peaks()
    exps = 2.0 * Hq * P
    mufu_peak = 16.0 * torch.cuda.get_device_properties(0).multi_processor_count * 1.965e9
    out = {"workload": pw["name"], "ms": ms,
           "tflops": flops / (ms / 1e3) / 1e12, "frac_of_bf16_peak": flops / (ms / 1e3) / 1e12 / bf16_peak,
           # K1 at 128K runs ~0.2 s of back-to-back tensor work: the sustained figure (cuBLAS run
           # back to back for 4 s, power-capped clocks) is the like-for-like denominator
           "frac_of_bf16_sustained": flops / (ms / 1e3) / 1e12 / bf16_sustained,
           "flop_count": "3 GEMM-eq = 6*d*L(L+1)/2 per q-head", "a_cumul_sum_over_G_lq": acs / (Hq * L),
           "exp_per_s": exps / (ms / 1e3), "exp_frac_of_mufu_peak": exps / (ms / 1e3) / mufu_peak,
           "exp_count": "2 per visible pair (pass 1 + A_cumul pass); MUFU peak 16/clk/SM at 1965 MHz, "
                        "a share of them evaluated on the FMA pipe (MKV_PREFILL_POLY)"}
    try:
        out["parity"] = prefill_parity(q, k, v, r, Hq, Hkv, L, d, scale, rows=(0, 4097, L // 2 + 3, L - 1),
                                       cols=[0, 1, 777, L // 3, L // 2, L - 130, L - 2, L - 1])
    except Exception as e:
        out["parity"] = {"error": repr(e)}
    hh = rw = int(math.floor(0.10 * L))
    ac = r.a_cumul.view(Hkv, L)
    cache = mkv.KVCache(Hkv, hh + rw, 0)
    kk, vv = k.view(Hkv, L, d), v.view(Hkv, L, d)
    kept, nk = mkv.select_token_counts(ac, hh, rw)
    cache.prefill_kept(kk, vv, kept, nk)
    torch.cuda.synchronize()
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
# driver
# ---------------------------------------------------------------------------
def spawn_ranks(args):
    """`bench.py --gpus N` outside torchrun: re-launch under torch.distributed.run, one rank per GPU."""
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def config_desc(args, world):
    W = WORKLOADS[args.workload]
    B = global_batch(args, world)
    return {"workload": W["desc"], "which": W["config_n1"] if world == 1 else W["config_multi"],
            "global_batch": B, "batch_per_gpu": B / world, "context": W["cfg"]["context"],
            "parallelism": f"dp{world} (sequence-batch shards via shard.plan, kv-heads split when B < N; "
                           f"no collective on the attention path)",
            "l2": "inputs larger than L2 (GBs of 2-bit pages per step vs 126 MB L2)"}


def reference_arm(args, world):
    """--impl reference: the reference's decode (oracle/_ref) on this host's cores, rank 0 only."""
    W = WORKLOADS[args.workload]
    cfg = W["cfg"]
    B = global_batch(args, world)
    threads = os.cpu_count() or 1
    upl = max(4, args.cpu_units_per_layer * 4)   # 16 units per layer: 512 of 4096 at configs[1]
    r = reference_decode(cfg, B, args.warmup + args.steps, 0, args.warmup, threads, upl)
    factor = r["units_total"] / r["units"]
    t_step = r["sample_step_s"] * factor
    value = B / t_step
    sample = (f"{r['units']} of {r['units_total']} (layer, seq, kv-head) units ({upl}/layer: every pyramid budget), "
              f"L={cfg['context']}, {args.steps} timed decode steps on {threads} threads; a full step's time = the "
              f"sample's measured step time x{factor:g} (units are independent, SPEC.md:144,401)")
    line = {"metric": W["metric"], "value": value, "unit": UNIT, "impl": "reference", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": r["sample_step_s"] * 1e3,
            "ms_per_step_note": "measured wall time of one sample step (steps x ms_per_step = the timed region); "
                                "value extrapolates it to the whole step",
            "extrapolation": {"units_timed": r["units"], "units_per_step": r["units_total"], "factor": factor,
                              "full_step_ms_extrapolated": t_step * 1e3},
            "higher_is_better": True, "scaling": "strong" if world > 1 else "weak", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic (integer-exact N(0,1) fp16 K/V, uniform A_cumul)",
            "config": config_desc(args, world),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference", "sample": sample,
                             "host": host_cpu()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    if not args.no_config0:
        try:
            import oracle
            c = CFG0
            hh = int(math.floor(c["alpha_hh"] * c["L"]))
            rw = int(math.floor(c["alpha_rw"] * c["L"]))
            rr = oracle.ref().pipeline_run(c["heads"], 1, c["L"], c["d"], hh, rw, c["steps"], SEED, threads)
            line["config0"] = {"workload": "configs[0] in full: 8 heads x (selective_flash_attn 4K -> prefill -> "
                                           "decode_step x 256)", "wall_s": rr["wall_s"], "threads": threads,
                               "decode_tokens_per_s_per_head": c["steps"] / (rr["decode_thread_s"] / c["heads"])}
        except Exception as e:
            line["config0"] = {"error": repr(e)}
    print(json.dumps(line))


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "reference":
        if rank == 0:
            reference_arm(args, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")) % max(torch.cuda.device_count(), 1))
        # NCCL for the barrier / max-over-ranks reduction; MKV_DIST_BACKEND=gloo lets several
        # ranks share one GPU (the 1-GPU validation of the N > 1 path)
        dist.init_process_group(os.environ.get("MKV_DIST_BACKEND", "nccl"))
    hbm_peak, bf16_peak, bf16_sust, peak_kind = load_peaks()
    W = WORKLOADS[args.workload]
    res = run_mkv(args, rank, world)
    threads = os.cpu_count() or 1
    extras = {}
    if rank == 0 and world == 1:
        cfg = W["cfg"]
        if not args.no_cpu_baseline:
            try:
                import oracle
                if oracle.ref_available():
                    r = reference_decode(cfg, global_batch(args, world), res["steps_total"], res["preroll"],
                                         args.warmup, threads, args.cpu_units_per_layer,
                                         compare=(res["last_out"], res["upl"]), one_thread_steps=2)
                    factor = r["units_total"] / r["units"]
                    B = global_batch(args, world)
                    extras["cpu_baseline"] = {
                        "value": B / (r["sample_step_s"] * factor), "unit": UNIT, "cores": threads,
                        "kind": "reference",
                        "sample": f"{r['units']} of {r['units_total']} (layer, seq, kv-head) units "
                                  f"({args.cpu_units_per_layer}/layer, every pyramid budget), {args.steps} timed decode "
                                  f"steps, {threads} threads; x{factor:g} to a full step (units are independent)",
                        "one_thread_value": B / (r["one_thread_step_s"] * factor),
                        "one_thread_sample_step_s": r["one_thread_step_s"], "sample_step_s": r["sample_step_s"],
                        "host": host_cpu()}
                    extras["parity"] = {
                        "what": "GPU decode outputs of the last timed step (mkv_decode_step_layers, 32 layers, through "
                                "the pre-roll and the in-window flush) vs the unmodified reference decode "
                                "(fp32 params) of the same units on the same synthetic streams",
                        "units": r["units"], "steps": res["steps_total"], "preroll_appends": res["preroll"],
                        "max_abs": r["max_abs"], "tol": DECODE_TOL, "ok": bool(r["max_abs"] <= DECODE_TOL)}
                else:
                    extras["cpu_baseline"] = {"unavailable": "oracle/_ref not built"}
            except Exception as e:
                extras["cpu_baseline"] = {"error": repr(e)}
        if not args.no_config0 and args.workload == "llama3-8b":
            try:
                extras["config0"] = config0(threads)
            except Exception as e:
                extras["config0"] = {"error": repr(e)}
        if not args.no_prefill:
            try:
                extras["prefill"] = run_prefill_bench(args)
                c0 = extras.get("config0") or {}
                one = (c0.get("cpu_reference") or {}).get("1")
                if one and "ms" in extras["prefill"]:
                    pw = W["prefill"]
                    flops = pw["hq"] * 6 * 128 * pw["L"] * (pw["L"] + 1) / 2
                    s1 = flops / (one["attn_gflops_per_thread"] * 1e9)
                    extras["prefill"]["cpu_reference"] = {
                        "kind": "reference", "extrapolated": True,
                        "how": "the reference selective_flash_attn's measured rate on configs[0]'s 8 x 4K heads "
                               "(config0.cpu_reference['1'].attn_gflops_per_thread; the work is 3 GEMM-eq "
                               "6 d L(L+1)/2 per head, so time scales quadratically in L)",
                        "seconds_1_thread": s1, "seconds_nproc": s1 / min(threads, pw["hq"]), "cores": threads,
                        "speedup_vs_gpu_nproc": s1 / min(threads, pw["hq"]) / (extras["prefill"]["ms"] / 1e3)}
            except Exception as e:  # reported, never silently substituted
                extras["prefill"] = {"error": repr(e)}
    if rank != 0:
        return
    kern = res["kernel"]
    traffic, traffic_src = load_traffic(kern["name"], kern["launch_units"]) if args.workload == "llama3-8b" and world == 1 else (None, None)
    line = {
        "metric": W["metric"], "value": res["tokens_per_s"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": res["ms_per_step"], "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None, "dtype": "fp16 (2-bit codes, fp16 params, fp32 accumulate)",
        "data": "synthetic (integer-exact N(0,1) fp16 K/V/q, uniform A_cumul), random-init shapes",
        "config": config_desc(args, world),
        "hbm_gbs": res["hbm_gbs"],
        "roofline": {"bound": "hbm", "achieved": kern["gbs"], "peak": hbm_peak, "unit": "GB/s",
                     "frac": kern["gbs"] / hbm_peak, "traffic": traffic, "traffic_source": traffic_src,
                     "kernel": kern["name"], "avg_launch_ms": kern["avg_launch_ms"],
                     "bytes_per_launch": kern["bytes_per_launch"], "launch_units": kern["launch_units"],
                     "peak_kind": peak_kind},
        "step_roofline_frac": res["hbm_gbs"] / (hbm_peak * world),
        "e2e": res["e2e"], "gpu_launches": res["gpu_launches"], "clocks": res["clocks"],
        "serving": res.get("serving"), "setup_s": res["setup_s"],
        "flushes_in_timed": res["flushes_in_timed"],
        "step_form": ("per layer: 32 page + 32 finish passes per step, layer l+1's page pass overlapping "
                      "layer l's merge (MKV_LAYERS_SPLIT)") if SPLIT else
                     ("every layer's q known up front: mkv_decode_step_layers over [32 layers x units] back to "
                      "back = one page pass + one finish pass over all units per step; 'serving' is the "
                      "dependent per-layer form"),
    }
    line.update({k: extras.get(k) for k in ("cpu_baseline", "parity", "config0", "prefill")})
    print(json.dumps(line))


if __name__ == "__main__":
    main()
