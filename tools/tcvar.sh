for v in A both; do cp paper_2411_18077_b200/lib_$v.so paper_2411_18077_b200/libminikv_b200.so; echo "== $v"; timeout 300 python -m pytest tests/test_gpu_decode.py -q -k "small" 2>&1 | tail -2; done
