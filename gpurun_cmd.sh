mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -p no:cacheprovider -k bench_config > gpurun_out/full6.log 2>&1; echo "rc $?" >> gpurun_out/full6.log
timeout 300 python scripts/attn_fwd_item_trace.py > gpurun_out/fwd_items.txt 2>&1
tail -3 gpurun_out/full6.log; cat gpurun_out/fwd_items.txt
