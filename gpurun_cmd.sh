timeout 300 python -m pytest tests/test_gpu_gemm.py -x -q 2>&1 | tail -2
for i in 1 2; do
echo NEW; timeout 120 python scripts/gemm_perf.py 2>&1 | grep -E "F proj|F fc1|F fc2|B fc2" | cut -c1-90
echo OLD; ZB_LIB=libzb_old.so timeout 120 python scripts/gemm_perf.py 2>&1 | grep -E "F proj|F fc1|F fc2|B fc2" | cut -c1-90
done
