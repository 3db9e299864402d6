mkdir -p gpurun_out
md5sum paper_2401_10241_b200/libzb.so > gpurun_out/c20_md5.txt
timeout 300 python -m pytest tests/test_gpu_attention.py tests/test_gpu_stage.py -q -x -p no:cacheprovider > gpurun_out/c20_tests.log 2>&1; echo "rc $?" >> gpurun_out/c20_tests.log
tail -3 gpurun_out/c20_tests.log
if grep -q "rc 0" gpurun_out/c20_tests.log; then
  timeout 300 python scripts/attn_perf.py > gpurun_out/c20_perf.jsonl 2>&1
  timeout 300 python scripts/attn_perf.py >> gpurun_out/c20_perf.jsonl 2>&1
  timeout 300 python scripts/attn_bwd_item_trace.py > gpurun_out/c20_bwd_items.txt 2>&1
  cat gpurun_out/c20_perf.jsonl gpurun_out/c20_bwd_items.txt
fi
