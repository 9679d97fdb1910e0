"""Time the fused K4 decode kernel on config-2-shaped layers (for ncu captures / A-B runs).

usage: python tools/decode_probe.py [n_layers] [residual_rows] [reps]
Builds n_layers of the Llama-3-8B 32K cache (pyramid budgets of the first n_layers
layers, B = 16, 8 kv-heads), appends residual_rows tokens, then times attend-only
launches and full decode steps (append + attend) with CUDA events.
"""
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2411_18077_b200 as mkv  # noqa: E402

NL = int(sys.argv[1]) if len(sys.argv) > 1 else 4
R = int(sys.argv[2]) if len(sys.argv) > 2 else 64
REPS = int(sys.argv[3]) if len(sys.argv) > 3 else 20
cfg = dict(bench.LLAMA, batch=16)
B, Hq, Hkv, d, L = cfg["batch"], cfg["n_q_heads"], cfg["n_kv_heads"], cfg["head_dim"], cfg["context"]
G = Hq // Hkv
hh, rw = bench.budgets(cfg)
upl = B * Hkv
cache = mkv.KVCache(NL * upl, [hh[l] + rw for l in range(NL) for _ in range(upl)], max_decode_tokens=R + 4 * REPS + 256)
for l in range(NL):
    u0 = l * upl
    k = mkv.synth_fp16((upl, L * d), 1, (2 << 48) | (u0 << 16), 1 << 16).view(upl, L, d)
    v = mkv.synth_fp16((upl, L * d), 1, (3 << 48) | (u0 << 16), 1 << 16).view(upl, L, d)
    a = mkv.synth_uniform((upl, L), 1, (7 << 48) | (u0 << 16), 1 << 16)
    cache.prefill(k, v, a, [hh[l]] * upl, rw, unit_begin=u0)
    del k, v, a
kn = mkv.synth_fp16((NL * upl, d), 1, 5 << 48, 1 << 16)
for _ in range(R):
    cache.append(kn, kn)
q = mkv.synth_fp16((NL, upl, G, d), 1, 4 << 48, 1 << 16)
out = torch.empty_like(q)
scale = 1 / math.sqrt(d)
torch.cuda.synchronize()
pages = sum(cache.unit_info(u)["n_pages"] for u in range(NL * upl))
byts = pages * 2048 + NL * upl * R * 4 * d + NL * upl * G * d * 4


from paper_2411_18077_b200 import _capi  # noqa: E402

att_args = (_capi.DecodeArgs * NL)()
stp_args = (_capi.DecodeArgs * NL)()
for l in range(NL):
    att_args[l] = _capi.DecodeArgs(l * upl, upl, G, q[l].data_ptr(), None, None, out[l].data_ptr(), scale)
    stp_args[l] = _capi.DecodeArgs(l * upl, upl, G, q[l].data_ptr(), kn[l * upl].data_ptr(), kn[l * upl].data_ptr(),
                                   out[l].data_ptr(), scale)
sp = int(torch.cuda.current_stream().cuda_stream)


def attend():  # one FFI crossing for all layers (host overhead off the GPU's critical path)
    _capi.check(_capi.lib().mkv_decode_step_layers(cache.h, NL, att_args, sp), "attend")


def step():
    _capi.check(_capi.lib().mkv_decode_step_layers(cache.h, NL, stp_args, sp), "step")


for fn, name in ((attend, "attend-only"), (step, "append+attend")):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(REPS):
        fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / (REPS * NL)
    print(f"{name}: {ms * 1e3:.2f} us/launch, {byts / NL / (ms / 1e3) / 1e9:.0f} GB/s (pages {pages}, R={R})")

if os.environ.get("MKV_DECODE_TRACE"):
    import numpy as np
    W = int(os.environ.get("MKV_PAGES_CFG", "8x2").split("x")[0])
    attend()  # one multi-layer call: the last two layers' timelines are in the two slots
    torch.cuda.synchronize()
    n = 2 * 4 * (148 * 12 + 8192)
    buf = np.zeros(n, np.uint64)
    got = _capi.lib().mkv_debug_decode_trace(cache.h, buf.ctypes.data, n)
    slot = got // 2
    pw = 4 * 148 * 12
    lay = []
    for sidx in range(2):
        t = buf[sidx * slot:(sidx + 1) * slot].astype(np.int64)
        pg = t[:pw].reshape(-1, 4)
        pg = pg[pg[:, 1] > 0]
        fn = t[pw:].reshape(-1, 4)
        fn = fn[fn[:, 0] > 0]
        lay.append((pg, fn))
    order = sorted(range(2), key=lambda i: lay[i][0][:, 0].min())
    t0 = lay[order[0]][0][:, 0].min()
    q_ = lambda a: " ".join(f"{(np.percentile(a, p) - t0) / 1e3:7.2f}" for p in (0, 50, 100))
    for name, i in (("layer n-2", order[0]), ("layer n-1", order[1])):
        pg, fn = lay[i]
        print(f"{name}: page kernel warps {len(pg)}, finish CTAs {len(fn)}   [us from layer n-2 start: min/median/max]")
        print("  pages start      ", q_(pg[:, 0]))
        print("  pages after wait ", q_(pg[:, 1]))
        print("  pages done       ", q_(pg[:, 2]))
        print("  finish start     ", q_(fn[:, 0]))
        print("  finish resid done", q_(fn[:, 1]))
        print("  finish wait rel. ", q_(fn[:, 2]))
        print("  finish end       ", q_(fn[:, 3]))
