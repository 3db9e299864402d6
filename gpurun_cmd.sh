mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_gemm.py -q -x -p no:cacheprovider -k "layernorm or bias" > gpurun_out/ln_fused_tests.log 2>&1; echo "rc $?" >> gpurun_out/ln_fused_tests.log
ZB_PDL=3 timeout 2400 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider > gpurun_out/gputests_pdl3.log 2>&1; echo "tests rc $?" >> gpurun_out/gputests_pdl3.log
ZB_PDL=3 timeout 1200 python bench.py --second-config none --no-cpu-baseline > gpurun_out/bench_lnfused_pdl3.log 2>&1
tail -5 gpurun_out/ln_fused_tests.log; tail -3 gpurun_out/gputests_pdl3.log; head -c 300 gpurun_out/bench_lnfused_pdl3.log
