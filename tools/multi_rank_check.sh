# N > 1 path of bench.py on one GPU: 2 ranks share it (gloo for the barrier / max-over-ranks)
export MKV_DIST_BACKEND=gloo
timeout 900 python bench.py --gpus 2 --steps 10 --warmup 3 --no-prefill > gpurun_out/mr_b2.json 2> gpurun_out/mr_b2.err; echo rc=$?
timeout 900 python bench.py --gpus 2 --batch 1 --steps 10 --warmup 3 --no-prefill > gpurun_out/mr_b2_headsplit.json 2> gpurun_out/mr_b2_headsplit.err; echo rc=$?
timeout 900 python bench.py --gpus 2 --workload lwm-7b --steps 6 --warmup 3 --no-prefill > gpurun_out/mr_lwm2.json 2> gpurun_out/mr_lwm2.err; echo rc=$?
