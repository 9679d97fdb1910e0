"""Timeline of the mma.sync page kernel (pages_kernel) from its per-warp globaltimer trace.

usage: MKV_DECODE_TRACE=1 python tools/k4_timeline.py [n_layers]
Builds n_layers of the Llama-3-8B 32K cache (configs[1] budgets, B = 16), then
  * one page pass alone (mkv_decode_pages_only, launched behind a synchronize): per-warp
    start, after-griddepcontrol.wait and done times relative to the first warp's start;
  * one multi-layer attend (mkv_decode_step_layers): the same for the last two layers.
Shows where a launch's time goes beyond the steady-state page rate: ramp (start spread,
first data), the tail (done spread), the gap between consecutive layers.
"""
import ctypes as C
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2411_18077_b200 as mkv  # noqa: E402
from paper_2411_18077_b200 import _capi  # noqa: E402

NL = int(sys.argv[1]) if len(sys.argv) > 1 else 4
cfg = bench.LLAMA
B, Hq, Hkv, d, L = 16, cfg["n_q_heads"], cfg["n_kv_heads"], cfg["head_dim"], cfg["context"]
G = Hq // Hkv
hh, rw = bench.budgets(cfg)
upl = B * Hkv
cache = mkv.KVCache(NL * upl, [hh[l] + rw for l in range(NL) for _ in range(upl)], max_decode_tokens=256)
for l in range(NL):
    u0 = l * upl
    k = mkv.synth_fp16((upl, L * d), 1, (2 << 48) | (u0 << 16), 1 << 16).view(upl, L, d)
    v = mkv.synth_fp16((upl, L * d), 1, (3 << 48) | (u0 << 16), 1 << 16).view(upl, L, d)
    a = mkv.synth_uniform((upl, L), 1, (7 << 48) | (u0 << 16), 1 << 16)
    cache.prefill(k, v, a, [hh[l]] * upl, rw, unit_begin=u0)
    del k, v, a
q = mkv.synth_fp16((NL, upl, G, d), 1, 4 << 48, 1 << 16)
tk = mkv.synth_fp16((NL, upl, d), 1, 5 << 48, 1 << 16)
out = torch.empty_like(q)
scale = 1 / math.sqrt(d)
for _ in range(3):
    cache.decode_step_layers(q, tk, tk, scale, out=out)
torch.cuda.synchronize()
sms = torch.cuda.get_device_properties(0).multi_processor_count
PAGE_WORDS = sms * max(4 * 12, 2 * 80)  # capi.cu trace_page_words()
SLOT = PAGE_WORDS + 4 * 8192
sp = int(torch.cuda.current_stream().cuda_stream)


def read_slots():
    buf = np.zeros(2 * SLOT, np.uint64)
    _capi.lib().mkv_debug_decode_trace(cache.h, buf.ctypes.data, 2 * SLOT)
    return [buf[s * SLOT:(s + 1) * SLOT].astype(np.int64) for s in range(2)]


def pct(a, t0):
    return " ".join(f"{(np.percentile(a, p) - t0) / 1e3:7.2f}" for p in (0, 10, 50, 90, 100))


# ---- one page pass alone ----
args = _capi.DecodeArgs(0, upl, G, q[0].data_ptr(), None, None, out[0].data_ptr(), scale)
for _ in range(2):
    _capi.check(_capi.lib().mkv_decode_pages_only(cache.h, C.byref(args), sp), "pages")
    torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
_capi.check(_capi.lib().mkv_decode_pages_only(cache.h, C.byref(args), sp), "pages")
e1.record()
torch.cuda.synchronize()
slots = read_slots()
best = max(slots, key=lambda t: int((t[:PAGE_WORDS].reshape(-1, 4)[:, 2] > 0).sum()))
pg = best[:PAGE_WORDS].reshape(-1, 4)[:sms * 8]
pg = pg[pg[:, 2] > 0]
t0 = pg[:, 0].min()
print(f"page pass alone: {e0.elapsed_time(e1) * 1e3:.1f} us by events; {len(pg)} warps "
      "[us from the first warp's start: min p10 median p90 max]")
print("  warp start       ", pct(pg[:, 0], t0))
print("  after wait       ", pct(pg[:, 1], t0))
print("  pages done       ", pct(pg[:, 2], t0))
print(f"  busy span (median done - median wait): {(np.median(pg[:, 2]) - np.median(pg[:, 1])) / 1e3:.2f} us")
busy = (pg[:, 2] - pg[:, 1]) / 1e3
for nseg in sorted(set(pg[:, 3].tolist())):
    m = pg[:, 3] == nseg
    print(f"  warps with {nseg} unit segment(s): {int(m.sum()):5d}, busy span median {np.median(busy[m]):6.2f} us, "
          f"max {np.max(busy[m]):6.2f} us")

# ---- a multi-layer attend: the last two layers ----
att = (_capi.DecodeArgs * NL)()
for l in range(NL):
    att[l] = _capi.DecodeArgs(l * upl, upl, G, q[l].data_ptr(), None, None, out[l].data_ptr(), scale)
_capi.check(_capi.lib().mkv_decode_step_layers(cache.h, NL, att, sp), "attend")
torch.cuda.synchronize()
slots = read_slots()
lays = []
for t in slots:
    p = t[:PAGE_WORDS].reshape(-1, 4)[:sms * 8]
    p = p[p[:, 2] > 0]
    f = t[PAGE_WORDS:].reshape(-1, 4)
    f = f[f[:, 0] > 0]
    if len(p):
        lays.append((p, f))
lays.sort(key=lambda x: x[0][:, 0].min())
t0 = lays[0][0][:, 0].min()
for name, (p, f) in zip(("layer n-2", "layer n-1"), lays):
    print(f"{name}: {len(p)} page warps, {len(f)} finish CTAs [us from layer n-2's first warp]")
    print("  pages start      ", pct(p[:, 0], t0))
    print("  pages after wait ", pct(p[:, 1], t0))
    print("  pages done       ", pct(p[:, 2], t0))
    if len(f):
        print("  finish start     ", pct(f[:, 0], t0))
        print("  finish resid done", pct(f[:, 1], t0))
        print("  finish wait rel. ", pct(f[:, 2], t0))
        print("  finish end       ", pct(f[:, 3], t0))

# ---- serving: one mkv_decode_step per layer, layer l+1's q = layer l's output ----
outs = torch.empty_like(q)
for _ in range(2):
    for l in range(NL):
        qp = q[0].data_ptr() if l == 0 else outs[l - 1].data_ptr()
        a = _capi.DecodeArgs(l * upl, upl, G, qp, None, None, outs[l].data_ptr(), scale)
        _capi.check(_capi.lib().mkv_decode_step(cache.h, C.byref(a), sp), "serve")
    torch.cuda.synchronize()
e0.record()
for l in range(NL):
    qp = q[0].data_ptr() if l == 0 else outs[l - 1].data_ptr()
    a = _capi.DecodeArgs(l * upl, upl, G, qp, None, None, outs[l].data_ptr(), scale)
    _capi.check(_capi.lib().mkv_decode_step(cache.h, C.byref(a), sp), "serve")
e1.record()
torch.cuda.synchronize()
print(f"serving: {NL} dependent layers in {e0.elapsed_time(e1) * 1e3:.1f} us by events "
      f"({e0.elapsed_time(e1) * 1e3 / NL:.1f} us per layer)")
slots = read_slots()
lays = []
for t in slots:
    p = t[:PAGE_WORDS].reshape(-1, 4)[:sms * 8]
    p = p[p[:, 2] > 0]
    f = t[PAGE_WORDS:].reshape(-1, 4)
    f = f[f[:, 0] > 0]
    lays.append((p, f))
lays.sort(key=lambda x: x[0][:, 0].min())
t0 = lays[0][0][:, 0].min()
for name, (p, f) in zip(("layer n-2", "layer n-1"), lays):
    print(f"{name}: {len(p)} page warps, {len(f)} finish CTAs [us from layer n-2's first warp]")
    print("  pages start      ", pct(p[:, 0], t0))
    print("  pages after wait ", pct(p[:, 1], t0))
    print("  pages done       ", pct(p[:, 2], t0))
    if len(f):
        print("  finish start     ", pct(f[:, 0], t0))
        print("  finish resid done", pct(f[:, 1], t0))
        print("  finish wait rel. ", pct(f[:, 2], t0))
        print("  finish end       ", pct(f[:, 3], t0))
    if len(f):
        fw = f[f[:, 0] >= t0]
        late = int((fw[:, 0] > p[:, 2].min()).sum())
        print(f"  finish CTAs of this layer (in window): {len(fw)}, started after its first page warp finished: {late}")
        print("  per CTA [us: min p10 median p90 max]")
        print("    residual attention ", pct(fw[:, 1] - fw[:, 0], 0))
        print("    wait release -> end", pct(fw[:, 3] - fw[:, 2], 0))
        print("    last page done -> wait release", pct(fw[:, 2] - p[:, 2].max(), 0))
