mkdir -p gpurun_out/abp
for cfg in 8x2 8x3 4x2 4x3; do
  MKV_PAGES_CFG=$cfg timeout 300 python bench.py --no-prefill --no-cpu-baseline --no-config0 > gpurun_out/abp/$cfg.json 2> gpurun_out/abp/$cfg.err
  python -c "
import json,sys; d=json.loads(open('gpurun_out/abp/$cfg.json').read().strip().splitlines()[-1])
print('$cfg', round(d['ms_per_step'],4), 'serving', round(d['serving']['ms_per_step'],4), 'pages', round(d['roofline']['avg_launch_ms'],4), 'e2e', round(d['e2e']['value']))
"
done
