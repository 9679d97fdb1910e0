"""mkv_cache_create time at configs[0]'s shape (8 units, 818 kept, 256 decode tokens) and at
configs[1]'s (4096 units), 10 creations each; MKV_PLAN_RESERVE=0 skips the all-units plan."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_18077_b200 as mkv  # noqa: E402

torch.cuda.init()
for n, cap in ((8, 818), (4096, 6000)):
    ts = []
    for _ in range(10):
        t0 = time.perf_counter()
        c = mkv.KVCache(n, cap, max_decode_tokens=384, n_r=128)
        ts.append((time.perf_counter() - t0) * 1e3)
        c.close()
    print(f"units {n}: create ms {' '.join(f'{t:.2f}' for t in ts)}")
