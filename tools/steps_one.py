"""configs[0]'s GPU chain once after a warm-up (for an ncu capture of steps_kernel):
    ncu --set full -k regex:steps_kernel -s 2 -c 1 python tools/steps_one.py"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import bench  # noqa: E402

r = bench.config0_gpu()
print({k: v for k, v in r["gpu_ms"].items()})
