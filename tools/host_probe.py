import time, math, sys, os
sys.path.insert(0, os.getcwd())
import torch
exec(open('tools/decode_probe.py').read().split("for fn, name in")[0])
import time
for fn, name in ((attend, "attend"), (step, "step")):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(REPS): fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"{name}: host issue {1e6*(t1-t0)/REPS:.1f} us per call ({NL} layers), wall incl. GPU {1e6*(t2-t0)/REPS:.1f} us per call")
