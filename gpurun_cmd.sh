timeout 600 python -m pytest tests/test_gpu_gemm.py -q -x --timeout 300 -p no:cacheprovider 2>&1 | tail -3
timeout 600 python scripts/gemm_w_bias.py 2>&1 | tail -12
