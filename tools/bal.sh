timeout 1800 python -m pytest tests/test_gpu_decode.py tests/test_gpu_mkvc.py -x -q 2>&1 | tail -2
for i in 1 2; do timeout 300 python bench.py --steps 20 --warmup 5 --no-prefill --no-cpu-baseline --no-config0 > gpurun_out/bal_b$i.json 2>gpurun_out/bal_b$i.err; done
timeout 300 python bench.py --workload lwm-7b --steps 10 --warmup 3 --no-prefill --no-cpu-baseline --no-config0 > gpurun_out/bal_lwm.json 2>gpurun_out/bal_lwm.err
