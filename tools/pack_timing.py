import math, sys, os, torch
sys.path.insert(0, os.getcwd())
import paper_2411_18077_b200 as mkv
Hkv, L, d = 8, 131072, 128
k = mkv.synth_fp16((Hkv, L, d), 1, 2 << 48, 1 << 16); v = mkv.synth_fp16((Hkv, L, d), 1, 3 << 48, 1 << 16)
a = mkv.synth_uniform((Hkv, L), 1, 7 << 48, 1 << 16)
for frac in (0.1, 0.25):
    hh = rw = int(frac * L)
    kept, nk = mkv.select_token_counts(a, hh, rw)
    cache = mkv.KVCache(Hkv, hh + rw, 0)
    cache.prefill_kept(k, v, kept, nk); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): cache.prefill_kept(k, v, kept, nk)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    by = Hkv * (hh + rw) * (4 * d + 4 + d)
    print(f"budget {2*frac:.1f}: pack {ms*1e3:.1f} us, {by/ms/1e6:.0f} GB/s")
    cache.close()
