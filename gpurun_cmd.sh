mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_gemm.py -q -x -p no:cacheprovider -k "layernorm" > gpurun_out/ln_fused_tests.log 2>&1; echo "rc $?" >> gpurun_out/ln_fused_tests.log
timeout 600 python scripts/gemm_ln_fused_perf.py > gpurun_out/r02_gemm_ln_fused_perf.jsonl 2>&1
ZB_PDL=3 timeout 1200 python bench.py --second-config none --no-cpu-baseline > gpurun_out/bench_lnfused2_pdl3.log 2>&1
tail -2 gpurun_out/ln_fused_tests.log; cat gpurun_out/r02_gemm_ln_fused_perf.jsonl; head -c 300 gpurun_out/bench_lnfused2_pdl3.log
