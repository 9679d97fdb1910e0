"""Per-step decode times over one residual cycle (a flush step included), config-2 shapes.

usage: python tools/flush_probe.py [n_layers] [steps]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.argv = [sys.argv[0], sys.argv[1] if len(sys.argv) > 1 else "32", "120", "1"] + sys.argv[2:]
src = open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "decode_probe.py")).read()
exec(src.split("for fn, name in")[0])  # cache with 120 residual rows, step() = append + attend
times = []
for s in range(16):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    step()
    e1.record()
    torch.cuda.synchronize()
    times.append(e0.elapsed_time(e1))
print(" ".join(f"{t:.3f}" for t in times))
print(f"flush step (8th) {times[7]:.3f} ms vs median {sorted(times)[8]:.3f} ms (each step synchronized)")

# the same 16 steps issued back to back (events between steps, one synchronize at the end):
# device time per step with the host running ahead, as in bench.py's timed loop
for s in range(200):  # advance to 7 steps before the next flush
    if cache.unit_info(0)["tokens_residual"] == cache.n_r - 8:
        break
    step()
torch.cuda.synchronize()
evs = [torch.cuda.Event(enable_timing=True) for _ in range(17)]
evs[0].record()
for s in range(16):
    step()
    evs[s + 1].record()
torch.cuda.synchronize()
dev = [evs[s].elapsed_time(evs[s + 1]) for s in range(16)]
print(" ".join(f"{t:.3f}" for t in dev))
print(f"flush step (8th) {dev[7]:.3f} ms vs median {sorted(dev)[8]:.3f} ms (back to back: device time)")

# split the flush cost: the append kernels alone (append-only call) and the next attend
# (which re-uploads the 32 changed plans)
for s in range(200):  # advance to one token before the next flush
    if all(cache.unit_info(u)["tokens_residual"] == cache.n_r - 1 for u in (0,)):
        break
    step()
torch.cuda.synchronize()
ts = []
for fn in (lambda: cache.append(kn, kn), attend, attend):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print(f"append-only flush {ts[0]:.3f} ms, first attend after it {ts[1]:.3f} ms (plan uploads), next attend {ts[2]:.3f} ms")
