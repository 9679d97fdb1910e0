"""Host cost of one mkv_decode_step call at configs[0]'s shape (8 units, G = 1, 818 kept + residual).

usage: python tools/step_call_probe.py [steps]
Prints, per decode step: host issue time through the Python wrapper (KVCache.decode_step, a
tensor slice per argument) and through the raw C ABI (prebuilt DecodeArgs), the device time of
the 256 steps issued back to back either way, and the steps kernel (mkv_decode_steps) for the
same stream.
"""
import ctypes as C
import math
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_18077_b200 as mkv  # noqa: E402
from paper_2411_18077_b200 import _capi  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 256
H, L, d, n_r = 8, 4096, 128, 128
hh = rw = int(math.floor(0.1 * L))
scale = 1.0 / math.sqrt(d)
k = mkv.synth_fp16((H, L * d), 7, 2 << 48, 1 << 16).view(H, L, d)
v = mkv.synth_fp16((H, L * d), 7, 3 << 48, 1 << 16).view(H, L, d)
a = torch.rand((H, L), device="cuda", dtype=torch.float32)
qd = mkv.synth_fp16((S, H * d), 7, 4 << 48, 1 << 16).view(S, H, 1, d)
kd = mkv.synth_fp16((S, H * d), 7, 5 << 48, 1 << 16).view(S, H, d)
vd = mkv.synth_fp16((S, H * d), 7, 6 << 48, 1 << 16).view(S, H, d)
outs = torch.empty_like(qd)
from paper_2411_18077_b200.ops import lib  # noqa: E402
L_ = lib()


def fresh():
    c = mkv.KVCache(H, hh + rw, max_decode_tokens=S + n_r, n_r=n_r)
    c.prefill(k, v, a, hh, rw)
    torch.cuda.synchronize()
    return c


def run(form):
    c = fresh()
    args = [_capi.DecodeArgs(0, H, 1, qd[s].data_ptr(), kd[s].data_ptr(), vd[s].data_ptr(), outs[s].data_ptr(), scale)
            for s in range(S)]
    sp = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    t0 = time.perf_counter()
    if form == "wrapper":
        for s in range(S):
            c.decode_step(qd[s], kd[s], vd[s], scale, out=outs[s])
    elif form == "capi":
        for s in range(S):
            _capi.check(L_.mkv_decode_step(c.h, C.byref(args[s]), sp), "decode")
    else:
        c.decode_steps(qd, kd, vd, scale, out=outs)
    host = (time.perf_counter() - t0) * 1e6 / S
    e1.record()
    torch.cuda.synchronize()
    dev = e0.elapsed_time(e1) * 1e3 / S
    c.close()
    return host, dev


for form in ("wrapper", "capi", "steps", "wrapper", "capi", "steps"):
    host, dev = run(form)
    print(f"{form:8s} host issue {host:6.2f} us/step, device {dev:6.2f} us/step")

# where the per-call host time goes: one entry point at a time, 2000 calls, host us per call
c = fresh()
sp = C.c_void_p(torch.cuda.current_stream().cuda_stream)
att = _capi.DecodeArgs(0, H, 1, qd[0].data_ptr(), None, None, outs[0].data_ptr(), scale)
N = 2000
x = torch.zeros(16, device="cuda")
for name, fn in (("torch x.add_(1) (reference launch)", lambda: x.add_(1)),
                 ("mkv_decode_pages_only", lambda: L_.mkv_decode_pages_only(c.h, C.byref(att), sp)),
                 ("mkv_decode_step attend-only", lambda: L_.mkv_decode_step(c.h, C.byref(att), sp)),
                 ("mkv_decode_step attend-only, sync each", lambda: (L_.mkv_decode_step(c.h, C.byref(att), sp),
                                                                   torch.cuda.synchronize()))):
    for _ in range(50):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(N):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"{name:40s} host {1e6 * (t1 - t0) / N:6.2f} us/call, wall {1e6 * (t2 - t0) / N:6.2f} us/call")
c.close()

# per-step host and wall times of the 256 append + attend calls (synchronized after each step)
c = fresh()
args = [_capi.DecodeArgs(0, H, 1, qd[s].data_ptr(), kd[s].data_ptr(), vd[s].data_ptr(), outs[s].data_ptr(), scale)
        for s in range(S)]
hs, ws = [], []
for s in range(S):
    t0 = time.perf_counter()
    _capi.check(L_.mkv_decode_step(c.h, C.byref(args[s]), sp), "decode")
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    hs.append(1e6 * (t1 - t0))
    ws.append(1e6 * (t2 - t0))
import numpy as np  # noqa: E402
hs, ws = np.array(hs), np.array(ws)
print(f"append+attend per step: host median {np.median(hs):.2f} us, max {hs.max():.1f} us at step {hs.argmax()}; "
      f"wall median {np.median(ws):.2f} us, max {ws.max():.1f} us at step {ws.argmax()}")
print("steps with host > 3x median:", [(int(i), round(float(hs[i]), 1)) for i in np.nonzero(hs > 3 * np.median(hs))[0]])
print("steps with wall > 2x median:", [(int(i), round(float(ws[i]), 1)) for i in np.nonzero(ws > 2 * np.median(ws))[0]])
c.close()

# the wrapper's current-stream lookup
for name, fn in (("torch.cuda.current_stream().cuda_stream", lambda: torch.cuda.current_stream().cuda_stream),
                 ("ops._stream_ptr()", lambda: mkv.ops._stream_ptr())):
    t0 = time.perf_counter()
    for _ in range(N):
        fn()
    print(f"{name:40s} {1e6 * (time.perf_counter() - t0) / N:6.2f} us/call")
