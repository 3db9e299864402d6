mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_attention.py tests/test_gpu_stage.py -q -x -p no:cacheprovider > gpurun_out/s16_tests.log 2>&1; echo "rc $?" >> gpurun_out/s16_tests.log
tail -3 gpurun_out/s16_tests.log
if grep -q "rc 0" gpurun_out/s16_tests.log; then
  timeout 300 python scripts/attn_perf.py > gpurun_out/s16_perf.jsonl 2>&1
  timeout 900 python bench.py --no-cpu-baseline > gpurun_out/s16_bench.log 2>&1; echo "rc $?" >> gpurun_out/s16_bench.log
  cat gpurun_out/s16_perf.jsonl; tail -c 300 gpurun_out/s16_bench.log
fi
