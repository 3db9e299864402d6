mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_attention.py -q -x -p no:cacheprovider > gpurun_out/c25_tests.log 2>&1; echo "rc $?" >> gpurun_out/c25_tests.log
tail -3 gpurun_out/c25_tests.log
if grep -q "rc 0" gpurun_out/c25_tests.log; then
  timeout 300 python scripts/attn_perf.py > gpurun_out/c25_perf.jsonl 2>&1
  timeout 300 python scripts/attn_perf.py >> gpurun_out/c25_perf.jsonl 2>&1
  timeout 300 python scripts/attn_cta_trace.py 3 1024 32 128 > gpurun_out/c25_cta.txt 2>&1
  timeout 300 python scripts/attn_cta_trace.py 6 1024 24 96 >> gpurun_out/c25_cta.txt 2>&1
  timeout 600 python -m pytest tests/test_gpu_stage.py tests/test_gpu_fullsize.py -q -x -p no:cacheprovider -k "not bench_config" > gpurun_out/c25_tests2.log 2>&1; echo "rc $?" >> gpurun_out/c25_tests2.log
  cat gpurun_out/c25_perf.jsonl gpurun_out/c25_cta.txt; tail -3 gpurun_out/c25_tests2.log
fi
