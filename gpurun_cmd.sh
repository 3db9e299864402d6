mkdir -p gpurun_out
timeout 150 python -m pytest tests/test_gpu_attention.py -q -x -p no:cacheprovider > gpurun_out/c28_tests.log 2>&1; echo "rc $?" >> gpurun_out/c28_tests.log
tail -3 gpurun_out/c28_tests.log
if grep -q "rc 0" gpurun_out/c28_tests.log; then
  timeout 300 python scripts/attn_perf.py > gpurun_out/c28_perf.jsonl 2>&1
  timeout 300 python scripts/attn_perf.py >> gpurun_out/c28_perf.jsonl 2>&1
  cat gpurun_out/c28_perf.jsonl
  timeout 900 python -m pytest tests/test_gpu_stage.py tests/test_gpu_pipeline_loopback.py -q -x -p no:cacheprovider > gpurun_out/c28_tests2.log 2>&1; echo "rc $?" >> gpurun_out/c28_tests2.log
  tail -3 gpurun_out/c28_tests2.log
fi
