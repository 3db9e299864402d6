timeout 900 python -m pytest tests/test_gpu_wgroup.py -q -x --timeout 600 -p no:cacheprovider 2>&1 | tail -15
timeout 600 python scripts/gemm_wgroup_perf.py 2>&1 | tail -10
