"""Small end-to-end run of every device path for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): K1 prefill (causal, GQA), K2 select, K3 pack (partial last page),
K4 decode through residual flushes (per step, multi-layer, decode_steps), the fp32
reference-format kernels, H2O.  Checks nothing numerically (the GPU suite does).

    compute-sanitizer --tool memcheck python tools/sanitize_small.py
"""
import math
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_2411_18077_b200 as mkv  # noqa: E402

torch.cuda.set_device(0)
d, Hq, Hkv, L = 128, 8, 2, 384
G = Hq // Hkv
scale = 1 / math.sqrt(d)
q = mkv.synth_fp16((1, Hq, L, d), 1, 1 << 48, 1 << 16)
k = mkv.synth_fp16((1, Hkv, L, d), 1, 2 << 48, 1 << 16)
v = mkv.synth_fp16((1, Hkv, L, d), 1, 3 << 48, 1 << 16)
r = mkv.selective_flash_attn(q, k, v, scale, True)
hh, rw = 37, 40  # 77 kept: partial last page
cache = mkv.KVCache(Hkv, hh + rw, max_decode_tokens=80, n_r=32)
cache.prefill(k[0], v[0], r.a_cumul[0], hh, rw)
S = 40  # crosses a flush (n_r = 32)
qd = mkv.synth_fp16((S, Hkv, G, d), 1, 4 << 48, 1 << 16)
kd = mkv.synth_fp16((S, Hkv, d), 1, 5 << 48, 1 << 16)
vd = mkv.synth_fp16((S, Hkv, d), 1, 6 << 48, 1 << 16)
for s in range(S // 2):
    cache.decode_step(qd[s], kd[s], vd[s], scale)
cache.decode_steps(qd[S // 2:], kd[S // 2:], vd[S // 2:], scale)
# two "layers" of one unit each, back to back: the coalesced multi-layer pass
c2 = mkv.KVCache(2, hh + rw, max_decode_tokens=40, n_r=32)
c2.prefill(k[0], v[0], r.a_cumul[0], hh, rw)
for s in range(34):
    c2.decode_step_layers(qd[s].view(2, 1, G, d), kd[s].view(2, 1, d), vd[s].view(2, 1, d), scale)
cache.check()
c2.check()
# fp32 reference-format kernels
q32, k32, v32 = (torch.randn(64, 32, device="cuda") for _ in range(3))
mkv.selective_flash_attn_f32(q32, k32, v32, 1 / math.sqrt(32), True)
mkv.decode_attention(q32[0], k32, v32, 1 / math.sqrt(32))
torch.cuda.synchronize()
print("sanitize_small: done")
