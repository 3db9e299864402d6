mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_attention.py -q -x -p no:cacheprovider > gpurun_out/c26_tests.log 2>&1; echo "rc $?" >> gpurun_out/c26_tests.log
tail -3 gpurun_out/c26_tests.log
timeout 300 python scripts/attn_perf.py > gpurun_out/c26_perf.jsonl 2>&1
timeout 300 python scripts/attn_perf.py >> gpurun_out/c26_perf.jsonl 2>&1
cat gpurun_out/c26_perf.jsonl
