"""Phase timeline of the tcgen05 page kernel (pages_tc_kernel) from its globaltimer trace.

usage: MKV_DECODE_TRACE=1 python tools/tc_trace.py [n_layers]
Builds n_layers of the Llama-3-8B 32K cache (configs[1] budgets, B = 16), runs one page pass
per layer with tracing, and prints the median duration of each phase of batches 4..7 over all
workers (compute warp 0 = the key-bias warp, compute warp 1, control warp).
"""
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2411_18077_b200 as mkv  # noqa: E402
from paper_2411_18077_b200 import _capi  # noqa: E402

NL = int(sys.argv[1]) if len(sys.argv) > 1 else 2
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
args = _capi.DecodeArgs(0, upl, G, q[0].data_ptr(), None, None, out[0].data_ptr(), scale)
sp = int(torch.cuda.current_stream().cuda_stream)
import ctypes as C  # noqa: E402
_capi.check(_capi.lib().mkv_decode_pages_only(cache.h, C.byref(args), sp), "pages")
torch.cuda.synchronize()
n = 1 << 20
buf = np.zeros(n, np.uint64)
got = _capi.lib().mkv_debug_decode_trace(cache.h, buf.ctypes.data, n)
slot = got // 2
W = 80
sms = torch.cuda.get_device_properties(0).multi_processor_count
best = None
for sidx in range(2):
    t = buf[sidx * slot: sidx * slot + 2 * sms * W].astype(np.int64).reshape(2 * sms, W)
    ok = t[:, 8] > 0
    if best is None or ok.sum() > best[1].sum():
        best = (t, ok)
t, ok = best
t = t[ok]
print(f"workers traced: {len(t)}")
names = ["full wait", "K extract + B_K (+Kb)", "V extract", "sFull wait", "softmax + p", "B_V + Vb + arrive",
         "epilogue/next"]
for wname, base in (("compute warp 0", 0), ("compute warp 1", 32)):
    print(wname + " (median ns per phase, batches 4..7):")
    for k in range(7):
        dur = [t[:, base + b * 8 + k + 1] - t[:, base + b * 8 + k] for b in range(4)]
        dur = np.concatenate(dur)
        print(f"  {names[k]:26s} {np.median(dur):8.0f}  p90 {np.percentile(dur, 90):8.0f}")
    per = [t[:, base + (b + 1) * 8] - t[:, base + b * 8] for b in range(3)]
    print(f"  batch period             {np.median(np.concatenate(per)):8.0f}")
print("control warp:")
cn = ["S issue (after opK)", "opV wait (after S issue)", "PV issue"]
for k in range(3):
    dur = np.concatenate([t[:, 64 + b * 4 + k + 1] - t[:, 64 + b * 4 + k] for b in range(4)])
    print(f"  {cn[k]:26s} {np.median(dur):8.0f}")
lat = np.concatenate([t[:, 0 + b * 8 + 4] - t[:, 64 + b * 4 + 1] for b in range(4)])
print(f"  S issued -> compute sees sFull {np.median(lat):8.0f}")
lat = np.concatenate([t[:, 64 + b * 4 + 0] - t[:, 0 + b * 8 + 2] for b in range(4)])
print(f"  compute arrives opK -> control sees it {np.median(lat):8.0f}")
