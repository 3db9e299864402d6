mkdir -p gpurun_out
ZB_ATTN_FWD=64 timeout 600 python -m pytest tests/test_gpu_attention.py -q -x -p no:cacheprovider --timeout 120 > gpurun_out/attn64_tests.log 2>&1; echo "rc $?" >> gpurun_out/attn64_tests.log
for v in 64 128 64; do ZB_ATTN_FWD=$v timeout 120 python scripts/attn_perf.py >> gpurun_out/r02_attn_perf_fwd64b.jsonl 2>&1; echo "# variant $v" >> gpurun_out/r02_attn_perf_fwd64b.jsonl; done
tail -3 gpurun_out/attn64_tests.log; cat gpurun_out/r02_attn_perf_fwd64b.jsonl
