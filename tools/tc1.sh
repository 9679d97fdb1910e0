set -x
timeout 300 python -m pytest tests/test_gpu_decode.py -x -q -k "small" 2>&1 | tail -15
timeout 600 python -m pytest tests/test_gpu_decode.py tests/test_gpu_mkvc.py -x -q 2>&1 | tail -15
timeout 300 python bench.py --steps 20 --warmup 5 --no-prefill --no-cpu-baseline --no-config0 > gpurun_out/tc_b1.json 2> gpurun_out/tc_b1.err; tail -3 gpurun_out/tc_b1.err
MKV_PAGES_IMPL=mma timeout 300 python bench.py --steps 20 --warmup 5 --no-prefill --no-cpu-baseline --no-config0 > gpurun_out/mma_b1.json 2> gpurun_out/mma_b1.err
