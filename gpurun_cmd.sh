mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_fullsize.py tests/test_gpu_stage.py -q -x -p no:cacheprovider > gpurun_out/attn_tests.log 2>&1; echo "rc $?" >> gpurun_out/attn_tests.log
timeout 300 python scripts/attn_perf.py > gpurun_out/r02_attn_perf_bwd_persistent.jsonl 2>&1
timeout 300 python scripts/attn_cta_trace.py 3 1024 32 128 > gpurun_out/r02_attn_cta_trace_p2.jsonl 2>&1
tail -3 gpurun_out/attn_tests.log; cat gpurun_out/r02_attn_perf_bwd_persistent.jsonl gpurun_out/r02_attn_cta_trace_p2.jsonl
