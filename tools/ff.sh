timeout 900 python -m pytest tests/test_gpu_decode.py tests/test_gpu_mkvc.py tests/test_gpu_select_quant.py tests/test_gpu_cpp_api.py -x -q 2>&1 | tail -3
echo "== fused"; timeout 300 python tools/flush_probe.py 32 2>&1 | head -2
echo "== launch"; MKV_FLUSH=launch timeout 300 python tools/flush_probe.py 32 2>&1 | head -2
timeout 300 python bench.py --steps 20 --warmup 5 --no-prefill --no-cpu-baseline --no-config0 > gpurun_out/ff_b.json 2>gpurun_out/ff_b.err; tail -2 gpurun_out/ff_b.err
MKV_FLUSH=launch timeout 300 python bench.py --steps 20 --warmup 5 --no-prefill --no-cpu-baseline --no-config0 > gpurun_out/ffl_b.json 2>gpurun_out/ffl_b.err
