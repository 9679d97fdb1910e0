# K3 A/B: staged builder (default) vs the round-1 gather builder (MKV_K3=gather); pack timing +
# one ncu capture of the staged kernel.  Run on the GPU box from the repo root.
out=${1:-gpurun_out/k3}
mkdir -p "$out"
python tools/pack_timing.py > "$out/staged.txt" 2>&1
MKV_K3=gather python tools/pack_timing.py > "$out/gather.txt" 2>&1
ncu --set full --clock-control none --import-source on -k regex:prefill_pages -s 2 -c 1 -o "$out/prof_k3" -f \
    python tools/pack_timing.py > /dev/null 2>&1
tail -n 20 "$out/staged.txt" "$out/gather.txt"
