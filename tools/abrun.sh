for v in "$@"; do
  if [ "$v" = base ]; then L=paper_2411_18077_b200/libminikv_b200.so; else L=abtest/$v/libminikv_b200.so; fi
  r=$(MKV_LIB_PATH=$L python bench.py --no-prefill --no-cpu-baseline --steps 64 --warmup 5 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.0f tok/s  %.4f ms/step  pages %.2f us  frac %.3f' % (d['value'], d['ms_per_step'], d['roofline']['avg_launch_ms']*1000, d['roofline']['frac']))")
  echo "$v: $r"
done
