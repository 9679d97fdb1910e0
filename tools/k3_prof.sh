cat > /tmp/k3.py <<'PY'
import math, sys, torch
sys.path.insert(0, '.')
import paper_2411_18077_b200 as mkv
Hkv, L, d = 8, 131072, 128
k = mkv.synth_fp16((Hkv, L, d), 1, 2 << 48, 1 << 16); v = mkv.synth_fp16((Hkv, L, d), 1, 3 << 48, 1 << 16)
a = mkv.synth_uniform((Hkv, L), 1, 7 << 48, 1 << 16)
for frac in (0.1, 0.5):
    hh = rw = int(frac / 2 * L)
    kept, nk = mkv.select_token_counts(a, hh, rw)
    c = mkv.KVCache(Hkv, hh + rw, 0)
    for _ in range(2): c.prefill_kept(k, v, kept, nk)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): c.prefill_kept(k, v, kept, nk)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"budget {frac}: {ms:.4f} ms, {Hkv*(hh+rw)*(4*d+4+d)/(ms/1e3)/1e9:.0f} GB/s")
    c.close()
PY
python /tmp/k3.py
ncu --set full --clock-control none --import-source on -k regex:prefill_pages -s 2 -c 1 -o gpurun_out/k3_prof -f python /tmp/k3.py > /dev/null 2>&1
echo done
