timeout 200 python -m pytest tests/test_gpu_ops.py -x -q 2>&1 | tail -1
for i in 1 2; do
echo NEW; timeout 100 python scripts/ops_perf.py 2>&1 | grep -E '"ln_fwd"|copy_bf16'
echo OLD; ZB_LIB=libzb_old.so timeout 100 python scripts/ops_perf.py 2>&1 | grep -E '"ln_fwd"'
done
