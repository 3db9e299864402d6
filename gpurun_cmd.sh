timeout 300 python -m pytest tests/test_gpu_gemm.py -x -q 2>&1 | tail -2
echo NEW; timeout 200 python scripts/gemm_epi_sweep.py 2>&1 | tail -10
echo OLD; ZB_LIB=libzb_old.so timeout 200 python scripts/gemm_epi_sweep.py 2>&1 | tail -10
