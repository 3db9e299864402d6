timeout 200 python scripts/gemm_epi_sweep.py 2>&1 | tail -10
timeout 200 python scripts/gemm_epi_sweep.py 6144 2304 9216 2>&1 | tail -10
