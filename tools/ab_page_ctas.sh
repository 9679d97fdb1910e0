# A/B of the page pass's CTA count (MKV_PAGE_CTAS; default one per SM): headline step, page launch,
# serving form.  Run on the GPU box from the repo root.
mkdir -p gpurun_out/abc
for n in 148 144 136 128 148; do
  MKV_PAGE_CTAS=$n timeout 300 python bench.py --no-prefill --no-cpu-baseline --no-config0 > gpurun_out/abc/$n.json 2> gpurun_out/abc/$n.err
  python -c "
import json; d=json.loads(open('gpurun_out/abc/$n.json').read().strip().splitlines()[-1])
print('$n', round(d['ms_per_step'],4), 'pages', round(d['roofline']['avg_launch_ms'],4), 'serving', round(d['serving']['ms_per_step'],4), 'e2e', round(d['e2e']['value']))
"
done
