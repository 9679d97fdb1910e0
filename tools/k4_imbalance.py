"""Per-warp busy time of one merged 32-layer page pass (configs[1], B = 16) against the warp's
unit-segment count: where the page kernel's tail (last warp done - median warp done) comes from.

usage: MKV_DECODE_TRACE=1 python tools/k4_imbalance.py
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

NL = 32
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
out = torch.empty_like(q)
scale = 1 / math.sqrt(d)
for _ in range(4):
    cache.decode_step_layers(q, None, None, scale, out=out)
torch.cuda.synchronize()
sms = torch.cuda.get_device_properties(0).multi_processor_count
PAGE_WORDS = sms * max(4 * 12, 2 * 80)
SLOT = PAGE_WORDS + 4 * 8192
buf = np.zeros(2 * SLOT, np.uint64)
_capi.lib().mkv_debug_decode_trace(cache.h, buf.ctypes.data, 2 * SLOT)
best = None
for s in range(2):
    t = buf[s * SLOT:s * SLOT + PAGE_WORDS].astype(np.int64).reshape(-1, 4)[:sms * 8]
    if best is None or t[:, 0].max() > best[:, 0].max():
        best = t
p = best[best[:, 2] > 0]
t0 = p[:, 1].min()
busy = (p[:, 2] - p[:, 1]) / 1e3
done = (p[:, 2] - t0) / 1e3
print(f"{len(p)} warps; done [us after the first wait release]: min {done.min():.1f} p10 {np.percentile(done, 10):.1f} "
      f"median {np.median(done):.1f} p90 {np.percentile(done, 90):.1f} max {done.max():.1f}")
for ns in sorted(set(p[:, 3].tolist())):
    m = p[:, 3] == ns
    print(f"  {ns} segments: {int(m.sum()):4d} warps, busy median {np.median(busy[m]):.1f} max {busy[m].max():.1f}")
wpc = 8
cta = np.arange(len(best))[best[:, 2] > 0] // wpc
per_cta = np.array([done[cta == c].max() for c in np.unique(cta)])
print(f"per CTA (SM) last warp done: min {per_cta.min():.1f} median {np.median(per_cta):.1f} max {per_cta.max():.1f}")
order = np.argsort(-per_cta)[:8]
print("slowest CTAs:", [(int(np.unique(cta)[i]), round(float(per_cta[i]), 1)) for i in order])
spread_in_cta = np.array([np.ptp(done[cta == c]) for c in np.unique(cta)])
print(f"spread of done times within a CTA: median {np.median(spread_in_cta):.1f} max {spread_in_cta.max():.1f} us")
