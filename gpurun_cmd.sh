mkdir -p gpurun_out
timeout 150 python -m pytest tests/test_gpu_attention.py -q -x -p no:cacheprovider > gpurun_out/c32_tests.log 2>&1; echo "rc $?" >> gpurun_out/c32_tests.log
tail -3 gpurun_out/c32_tests.log
if grep -q "rc 0" gpurun_out/c32_tests.log; then
  timeout 300 python scripts/attn_perf.py > gpurun_out/c32_perf.jsonl 2>&1
  timeout 300 python scripts/attn_perf.py >> gpurun_out/c32_perf.jsonl 2>&1
  timeout 300 python scripts/attn_fwd_trace.py > gpurun_out/c32_blocks.txt 2>&1
  cat gpurun_out/c32_perf.jsonl gpurun_out/c32_blocks.txt
fi
