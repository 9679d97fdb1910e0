for c in 148 144 140 136 128; do MKV_PAGE_CTAS=$c timeout 300 python bench.py --steps 40 --warmup 5 --no-prefill --no-cpu-baseline --no-config0 > gpurun_out/bal2_$c.json 2>/dev/null; done
