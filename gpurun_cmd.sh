timeout 60 python scripts/gemm_trace.py 6144 9216 2304 1 3 2>&1 | tail -16
timeout 60 python scripts/gemm_trace.py 6144 9216 2304 1 0 2>&1 | tail -16
