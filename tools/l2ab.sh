for i in 1 2; do timeout 300 python bench.py --steps 40 --warmup 5 --no-prefill --no-cpu-baseline --no-config0 > gpurun_out/l2_$i.json 2>gpurun_out/l2_$i.err; done
timeout 300 python bench.py --steps 20 --warmup 5 --no-prefill --no-cpu-baseline --no-config0 > gpurun_out/l2_20.json 2>/dev/null
