timeout 60 python -m pytest tests/test_gpu_attention.py -x -q 2>&1 | tail -2
timeout 60 python scripts/attn_perf.py 2>&1 | tail -3
