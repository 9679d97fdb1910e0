#!/bin/bash
# Round profiling pass (run on the GPU box from the repo root):
#   1. the bench line (N=1) and the reference arm,  2. the ncu launch list of a short bench run,
#   3. per-launch DRAM traffic of the K4 page kernel (one launch per step over all 32 layers'
#      units; roofline "traffic"),
#   4. one --set full capture each of pages_kernel, finish_kernel and the K1 prefill kernels.
set -u
out=${1:-gpurun_out}
mkdir -p "$out"
python bench.py > "$out/bench.json" 2> "$out/bench.err"
python bench.py --impl reference > "$out/bench_ref.json" 2> "$out/bench_ref.err"
SHORT="--steps 2 --warmup 3 --no-prefill --no-cpu-baseline --no-config0 --no-serving"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$out/launches.csv" \
    python bench.py $SHORT > /dev/null 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:'^pages_kernel' -s 3 -c 4 --csv --log-file "$out/pages_traffic.csv" \
    python bench.py $SHORT > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:'^pages_kernel' -s 4 -c 1 -o "$out/prof_pages" -f \
    python bench.py $SHORT > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:finish_kernel -s 4 -c 1 -o "$out/prof_finish" -f \
    python bench.py $SHORT > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:attn_fwd_kernel -s 1 -c 1 -o "$out/prof_fwd" -f \
    python tools/prefill_one.py 16384 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:acumul_kernel -s 1 -c 1 -o "$out/prof_acum" -f \
    python tools/prefill_one.py 16384 > /dev/null 2>&1
echo profile done
