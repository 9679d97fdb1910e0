for cfg in 8x2 4x2 4x3; do MKV_PAGES_CFG=$cfg timeout 300 python bench.py --steps 40 --warmup 5 --no-prefill --no-cpu-baseline --no-config0 > gpurun_out/cfg_$cfg.json 2>gpurun_out/cfg_$cfg.err; done
