timeout 600 python -m pytest tests/test_gpu_decode.py -x -q 2>&1 | tail -2
timeout 300 python bench.py --steps 20 --warmup 5 --no-prefill --no-cpu-baseline --no-config0 > gpurun_out/tc4_b1.json 2> gpurun_out/tc4_b1.err
MKV_DECODE_TRACE=1 timeout 300 python tools/tc_trace.py 2
