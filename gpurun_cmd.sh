mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_attention.py -q -x -p no:cacheprovider > gpurun_out/c35_tests.log 2>&1; echo "rc $?" >> gpurun_out/c35_tests.log
tail -3 gpurun_out/c35_tests.log
if grep -q "rc 0" gpurun_out/c35_tests.log; then
  for lib in libzb.so libzb_nohint.so libzb.so libzb_nohint.so; do
    echo "# $lib" >> gpurun_out/c35_perf.jsonl
    ZB_LIB=$lib timeout 300 python scripts/attn_perf.py >> gpurun_out/c35_perf.jsonl 2>&1
    ZB_LIB=$lib timeout 300 python scripts/gemm_b_layout.py --secs 0.5 >> gpurun_out/c35_perf.jsonl 2>&1
  done
  for lib in libzb.so libzb_nohint.so libzb.so libzb_nohint.so; do
    echo "# $lib" >> gpurun_out/c35_bench.txt
    ZB_LIB=$lib timeout 600 python bench.py --second-config none --no-profile-p8 --no-cpu-baseline --no-e2e > gpurun_out/c35_b.log 2>&1
    python -c "
import json
for l in open('gpurun_out/c35_b.log'):
    if l.startswith('{'):
        d=json.loads(l); print(json.dumps({'value': d['value'], 'mhz': d['clocks']['sm_mhz'], 'gemm': d['roofline']['achieved'], 'cls': {k: round(v['tflops'],1) for k,v in d['roofline']['per_class'].items()}}))
" >> gpurun_out/c35_bench.txt
  done
  cat gpurun_out/c35_perf.jsonl gpurun_out/c35_bench.txt
fi
