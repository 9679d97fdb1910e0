import math, torch, sys
sys.path.insert(0, '.')
import paper_2411_18077_b200 as mkv
for (B, Hq, Hkv, L) in [(1, 32, 8, 4096), (1, 32, 8, 16384), (1, 32, 8, 32768)]:
    q = mkv.synth_fp16((B, Hq, L, 128), 1, 1 << 48, 1 << 16); k = mkv.synth_fp16((B, Hkv, L, 128), 1, 2 << 48, 1 << 16); v = mkv.synth_fp16((B, Hkv, L, 128), 1, 3 << 48, 1 << 16)
    for _ in range(3): r = mkv.selective_flash_attn(q, k, v, 1 / math.sqrt(128), True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3): r = mkv.selective_flash_attn(q, k, v, 1 / math.sqrt(128), True)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    fl = Hq * 6 * 128 * L * (L + 1) / 2 * B
    print(f"L={L} ms={ms:.3f} TFLOP/s(3-GEMM)={fl/ms/1e9:.1f} sum/(G*L)={r.a_cumul.double().sum().item()/(Hq*L):.6f}")
