mkdir -p gpurun_out
for c in 296 592 888 1184 296 592; do echo "# ZB_COLRED_CTAS=$c" >> gpurun_out/colred.jsonl; ZB_COLRED_CTAS=$c timeout 300 python scripts/ln_fwd_perf.py >> gpurun_out/colred.jsonl 2>&1; done
cat gpurun_out/colred.jsonl
