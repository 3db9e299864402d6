timeout 60 python -m pytest tests/test_gpu_attention.py -x -q 2>&1 | tail -2
for i in 1 2; do timeout 60 python scripts/attn_perf.py 2>&1 | tail -3 | cut -c1-60; done
