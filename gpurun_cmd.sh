timeout 60 python scripts/attn_perf.py 2>&1 | tail -3 > gpurun_out/attn_perf_r2.jsonl; cat gpurun_out/attn_perf_r2.jsonl
timeout 60 ./scripts/micro/mma_rate > gpurun_out/mma_rate.txt 2>&1; timeout 60 ./scripts/micro/mma_issue > gpurun_out/mma_issue.txt 2>&1; timeout 60 ./scripts/micro/ex2_rate > gpurun_out/ex2_rate.txt 2>&1
