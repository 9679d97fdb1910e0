import torch, time
for mb in (1, 6, 64):
    n = mb * 1024 * 1024 // 2
    h = torch.empty(n, dtype=torch.float16).pin_memory()
    d = torch.empty(n, dtype=torch.float16, device='cuda')
    s = torch.cuda.Stream()
    for direction in ('h2d', 'd2h'):
        with torch.cuda.stream(s):
            for _ in range(3):
                (d.copy_(h, non_blocking=True) if direction == 'h2d' else h.copy_(d, non_blocking=True))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(10):
                (d.copy_(h, non_blocking=True) if direction == 'h2d' else h.copy_(d, non_blocking=True))
            e1.record(s)
        s.synchronize()
        ms = e0.elapsed_time(e1) / 10
        print(f"{direction} {mb} MB: {ms*1e3:.0f} us  {mb/1024/(ms/1e3):.1f} GB/s")
