mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_stage.py tests/test_gpu_fullsize.py -q -x -p no:cacheprovider -k "not c4_c5" > gpurun_out/c38_tests.log 2>&1; echo "rc $?" >> gpurun_out/c38_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/c38_smoke.log 2>&1; echo "rc $?" >> gpurun_out/c38_smoke.log
timeout 300 python scripts/attn_perf.py > gpurun_out/c38_perf.jsonl 2>&1
tail -2 gpurun_out/c38_tests.log; tail -2 gpurun_out/c38_smoke.log; cat gpurun_out/c38_perf.jsonl
