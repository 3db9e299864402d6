mkdir -p gpurun_out
timeout 600 python scripts/gemm_b_layout.py --secs 1.0 > gpurun_out/b_layout.jsonl 2>&1
timeout 600 python scripts/gemm_b_layout.py --secs 1.0 >> gpurun_out/b_layout.jsonl 2>&1
cat gpurun_out/b_layout.jsonl
