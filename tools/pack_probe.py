"""Time K3 (gather + 2-bit quantize + pack) at configs[3]'s shape (8 kv-head units of a 128K
prompt, 20% budget) and configs[1]'s (128 units of 32K, pyramid layer-0 budget); for ncu."""
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_18077_b200 as mkv  # noqa: E402

for n, L, hh, rw in ((8, 131072, 13107, 13107), (128, 32768, 6084, 3276)):
    d = 128
    k = mkv.synth_fp16((n, L * d), 1, 2 << 48, 1 << 16).view(n, L, d)
    v = mkv.synth_fp16((n, L * d), 1, 3 << 48, 1 << 16).view(n, L, d)
    a = mkv.synth_uniform((n, L), 1, 7 << 48, 1 << 16)
    kept, nk = mkv.select_token_counts(a, hh, rw)
    cache = mkv.KVCache(n, hh + rw, 0)
    for _ in range(2):
        cache.prefill_kept(k, v, kept, nk)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        cache.prefill_kept(k, v, kept, nk)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    byts = n * (hh + rw) * (4 * d + 4 + d)
    print(f"K3 {n} x {L}: {ms:.3f} ms, {byts / ms / 1e6:.0f} GB/s")
    cache.close()
    del k, v, a
