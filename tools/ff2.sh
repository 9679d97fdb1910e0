timeout 1800 python -m pytest tests/test_gpu_decode.py tests/test_gpu_mkvc.py -x -q 2>&1 | tail -3
echo "== default"; timeout 300 python tools/flush_probe.py 32 2>&1 | head -2
echo "== fused"; MKV_FLUSH=fused timeout 300 python tools/flush_probe.py 32 2>&1 | head -2
for i in 1 2; do timeout 300 python bench.py --steps 20 --warmup 5 --no-prefill --no-cpu-baseline --no-config0 > gpurun_out/ff2_b$i.json 2>gpurun_out/ff2_b$i.err; done
MKV_FLUSH=fused timeout 300 python bench.py --steps 20 --warmup 5 --no-prefill --no-cpu-baseline --no-config0 > gpurun_out/ff2_f.json 2>gpurun_out/ff2_f.err
