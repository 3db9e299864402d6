timeout 300 python -m pytest tests/test_gpu_attention.py -x -q -m gpu 2>&1 | tail -15
echo "=== tc"; timeout 200 python scripts/attn_perf.py 2>&1 | tail -4
