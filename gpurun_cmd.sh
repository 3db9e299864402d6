mkdir -p gpurun_out
timeout 300 python scripts/attn_fwd_item_trace.py > gpurun_out/fwd_items_end.txt 2>&1
timeout 300 python scripts/attn_fwd_trace.py > gpurun_out/fwd_blocks_end.txt 2>&1
cat gpurun_out/fwd_items_end.txt gpurun_out/fwd_blocks_end.txt
