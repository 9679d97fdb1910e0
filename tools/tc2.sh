set -x
timeout 600 python -m pytest tests/test_gpu_decode.py tests/test_gpu_mkvc.py -x -q 2>&1 | tail -5
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pages_tc -s 64 -c 1 -o gpurun_out/tc_prof -f python bench.py --steps 2 --warmup 3 --no-prefill --no-cpu-baseline --no-config0 --no-serving > gpurun_out/tc_ncu.log 2>&1; tail -3 gpurun_out/tc_ncu.log
