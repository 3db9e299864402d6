mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_attention.py -q -x -p no:cacheprovider > gpurun_out/tma_tests.log 2>&1; echo "rc $?" >> gpurun_out/tma_tests.log
tail -3 gpurun_out/tma_tests.log
if grep -q "rc 0" gpurun_out/tma_tests.log; then
  timeout 300 python scripts/attn_perf.py > gpurun_out/tma_perf.jsonl 2>&1
  timeout 300 python scripts/attn_perf.py >> gpurun_out/tma_perf.jsonl 2>&1
  timeout 300 python scripts/attn_bwd_item_trace.py > gpurun_out/bwd_items_tma.txt 2>&1
  cat gpurun_out/tma_perf.jsonl gpurun_out/bwd_items_tma.txt
fi
