timeout 600 python -m pytest tests/test_gpu_decode.py -x -q 2>&1 | tail -2
for i in 1 2; do timeout 300 python bench.py --steps 20 --warmup 5 --no-prefill --no-cpu-baseline --no-config0 > gpurun_out/tc3_b$i.json 2> gpurun_out/tc3_b$i.err; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pages_tc -s 64 -c 1 -o gpurun_out/tc3_prof -f python bench.py --steps 2 --warmup 3 --no-prefill --no-cpu-baseline --no-config0 --no-serving > gpurun_out/tc3_ncu.log 2>&1
