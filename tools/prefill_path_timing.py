"""Time K2 (select) and K3 (gather + 2-bit pack) for config-4 budgets (Mistral-7B 128K, 8 kv-heads)
and for one config-2 layer (Llama-3-8B, 32K, B=16)."""
import math, sys, time, torch
sys.path.insert(0, '.')
import paper_2411_18077_b200 as mkv

def run(n_units, L, hh, rw, label):
    d = 128
    k = mkv.synth_fp16((n_units, L * d), 1, 2 << 48, 1 << 16).view(n_units, L, d)
    v = mkv.synth_fp16((n_units, L * d), 1, 3 << 48, 1 << 16).view(n_units, L, d)
    a = mkv.synth_uniform((n_units, L), 1, 7 << 48, 1 << 16)
    cache = mkv.KVCache(n_units, hh + rw, 0)
    for _ in range(2): cache.prefill(k, v, a, hh, rw)
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record()
    for _ in range(5): kept, nk = mkv.select_token_counts(a, hh, rw)
    e[1].record()
    for _ in range(5): cache.prefill_kept(k, v, kept, nk)
    e[2].record(); torch.cuda.synchronize()
    t_sel = e[0].elapsed_time(e[1]) / 5
    t_pre = e[1].elapsed_time(e[2]) / 5
    n_kept = min(hh + rw, L)
    sel_bytes = n_units * (4 * L + 4 * n_kept)
    quant_bytes = n_units * n_kept * (4 * d + 4 + d)
    print(f"{label}: K2 select {t_sel*1e3:.1f} us ({sel_bytes/t_sel/1e6:.0f} GB/s)   K3 gather+pack {t_pre*1e3:.1f} us "
          f"({quant_bytes/t_pre/1e6:.0f} GB/s)")

for frac in (0.1, 0.2, 0.3, 0.4, 0.5):
    L = 131072
    run(8, L, int(L * frac / 2), int(L * frac / 2), f"cfg4 budget {int(frac*100)}%")
run(128, 32768, 6084, 3276, "cfg2 layer 0")
