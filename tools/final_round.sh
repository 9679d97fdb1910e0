#!/bin/bash
# Round-end evidence pass on the GPU box (repo root): GPU suite + smoke, compute-sanitizer over
# every device path (default finish form and the forced split form), then tools/profile_round.sh
# (bench line, reference arm, launch list, page-kernel traffic, ncu --set full captures).
set -u
out=${1:-gpurun_out/final}
mkdir -p "$out"
timeout 1500 python -m pytest tests -m gpu -q > "$out/gpu_tests.txt" 2>&1; tail -3 "$out/gpu_tests.txt"
python -c "import __graft_entry__ as g; g.smoke()" > "$out/smoke.txt" 2>&1; echo "smoke rc=$?"
for mode in default split; do
  for tool in memcheck racecheck synccheck initcheck; do
    echo "## $tool ($mode)" >> "$out/sanitizer.txt"
    if [ $mode = split ]; then export MKV_MERGE=split; else unset MKV_MERGE; fi
    timeout 900 compute-sanitizer --tool $tool python tools/sanitize_small.py >> "$out/sanitizer.txt" 2>&1
    unset MKV_MERGE
  done
done
grep -E "SUMMARY|##" "$out/sanitizer.txt"
bash tools/profile_round.sh "$out"
timeout 900 python bench.py --workload lwm-7b > "$out/bench_lwm.json" 2> "$out/bench_lwm.err"; echo "lwm rc=$?"
bash tools/multi_rank_check.sh > "$out/multirank.txt" 2>&1
for f in mr_b2 mr_b2_headsplit mr_lwm2; do echo "== $f" >> "$out/multirank.txt"; tail -1 gpurun_out/$f.json >> "$out/multirank.txt"; done
