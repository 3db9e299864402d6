timeout 300 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_stage.py -x -q -m gpu 2>&1 | tail -5
echo "=== 2CTA 8 epi warps"; timeout 200 python scripts/gemm_perf.py 2>&1 | tail -12
