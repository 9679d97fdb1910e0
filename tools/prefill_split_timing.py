"""Per-kernel K1 times (attn_fwd_kernel = pass 1, acumul_kernel = pass 2) from CUPTI kernel
records (torch.profiler), at Mistral-7B layer shapes (32 q / 8 kv heads, d = 128, causal).

    python tools/prefill_split_timing.py [L ...]

Rates are in each pass's own GEMM-equivalents: pass 1 = 4 d P per q-head (QK^T + PV), pass 2 =
2 d P (the QK^T recompute), P = L (L + 1) / 2; fractions against MEASURED_PEAKS.json's burst
bf16 figure.  MKV_PREFILL_POLY selects the exponential split (see prefill.cu)."""
import json
import math
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_2411_18077_b200 as mkv  # noqa: E402

try:
    peak = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["bf16_tflops"]
except Exception:
    peak = 1590.0
Ls = [int(a) for a in sys.argv[1:]] or [16384, 131072]
Hq, Hkv, d = 32, 8, 128
for L in Ls:
    q = mkv.synth_fp16((1, Hq, L, d), 1, 1 << 48, 1 << 16)
    k = mkv.synth_fp16((1, Hkv, L, d), 1, 2 << 48, 1 << 16)
    v = mkv.synth_fp16((1, Hkv, L, d), 1, 3 << 48, 1 << 16)
    for _ in range(2):
        r = mkv.selective_flash_attn(q, k, v, 1 / math.sqrt(d), True)
    torch.cuda.synchronize()
    reps = 3 if L <= 65536 else 2
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(reps):
            r = mkv.selective_flash_attn(q, k, v, 1 / math.sqrt(d), True)
        torch.cuda.synchronize()
    t = {}
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA:
            for name, key in (("attn_fwd", "attn_fwd_kernel"), ("acumul_kernel", "acumul_kernel")):
                if name in e.name:
                    t.setdefault(key, []).append(e.device_time_total / 1e3)  # us -> ms
    P = L * (L + 1) / 2
    f1, f2 = Hq * 4 * d * P, Hq * 2 * d * P
    a, b = min(t["attn_fwd_kernel"]), min(t["acumul_kernel"])
    s = r.a_cumul.double().sum().item() / (Hq * L)
    print(json.dumps({"L": L, "poly": os.environ.get("MKV_PREFILL_POLY", "default"),
                      "fwd_ms": round(a, 3), "fwd_tflops": round(f1 / a / 1e9, 1), "fwd_frac": round(f1 / a / 1e9 / peak, 3),
                      "acumul_ms": round(b, 3), "acumul_tflops": round(f2 / b / 1e9, 1),
                      "acumul_frac": round(f2 / b / 1e9 / peak, 3),
                      "k1_frac": round((f1 + f2) / (a + b) / 1e9 / peak, 3), "sum_over_GL": round(s, 7)}))
    del q, k, v, r
    torch.cuda.empty_cache()
