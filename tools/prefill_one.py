"""One K1 prefill call at a given shape (for ncu captures)."""
import math, sys, torch
sys.path.insert(0, '.')
import paper_2411_18077_b200 as mkv
L = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
Hq, Hkv = 32, 8
q = mkv.synth_fp16((1, Hq, L, 128), 1, 1 << 48, 1 << 16); k = mkv.synth_fp16((1, Hkv, L, 128), 1, 2 << 48, 1 << 16)
v = mkv.synth_fp16((1, Hkv, L, 128), 1, 3 << 48, 1 << 16)
for _ in range(2):
    r = mkv.selective_flash_attn(q, k, v, 1 / math.sqrt(128), True)
torch.cuda.synchronize()
