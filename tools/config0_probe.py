import math, time, sys, os
sys.path.insert(0, os.getcwd())
import torch
import paper_2411_18077_b200 as mkv
H, L, d, steps = 8, 4096, 128, 256
hh = rw = 409
q = mkv.synth_fp16((H, L * d), 1, 1 << 48, 1 << 16).view(1, H, L, d)
k = mkv.synth_fp16((H, L * d), 1, 2 << 48, 1 << 16).view(1, H, L, d)
v = mkv.synth_fp16((H, L * d), 1, 3 << 48, 1 << 16).view(1, H, L, d)
qd = torch.stack([mkv.synth_fp16((H, d), 1, (4 << 48) | (s + 1), 1 << 16) for s in range(steps)]).view(steps, H, 1, d)
kd = torch.stack([mkv.synth_fp16((H, d), 1, (5 << 48) | (s + 1), 1 << 16) for s in range(steps)])
vd = torch.stack([mkv.synth_fp16((H, d), 1, (6 << 48) | (s + 1), 1 << 16) for s in range(steps)])
outs = torch.empty((steps, H, 1, d), dtype=torch.float16, device="cuda")
scale = 1 / math.sqrt(d)
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    cache = mkv.KVCache(H, hh + rw, max_decode_tokens=steps + 128, n_r=128)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    r = mkv.selective_flash_attn(q, k, v, scale, True)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    cache.prefill(k[0], v[0], r.a_cumul[0], hh, rw)
    torch.cuda.synchronize(); t3 = time.perf_counter()
    for s in range(steps):
        cache.decode_step(qd[s], kd[s], vd[s], scale, out=outs[s])
    t4 = time.perf_counter()
    torch.cuda.synchronize(); t5 = time.perf_counter()
    qs = [qd[s] for s in range(steps)]; ks_ = [kd[s] for s in range(steps)]; vs_ = [vd[s] for s in range(steps)]; os_ = [outs[s] for s in range(steps)]
    cache.close()
    print(f"make_cache {1e3*(t1-t0):.2f} attn {1e3*(t2-t1):.2f} prefill {1e3*(t3-t2):.2f} decode host-issue {1e3*(t4-t3):.2f} decode total {1e3*(t5-t3):.2f} ms")

# CUPTI view of one chain: device kernels and the runtime API calls the host spends its time in
from torch.profiler import ProfilerActivity, profile
cache = mkv.KVCache(H, hh + rw, max_decode_tokens=steps + 128, n_r=128)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    r = mkv.selective_flash_attn(q, k, v, scale, True)
    cache.prefill(k[0], v[0], r.a_cumul[0], hh, rw)
    for s in range(16):
        cache.decode_step(qd[s], kd[s], vd[s], scale, out=outs[s])
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="self_cpu_time_total", row_limit=25))
