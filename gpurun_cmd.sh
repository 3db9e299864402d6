mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_stage.py tests/test_gpu_ops.py -x -q -p no:cacheprovider > gpurun_out/t3.log 2>&1; echo "rc $?" >> gpurun_out/t3.log
for v in 0 1 0 1; do ZB_LN_FWD=$v timeout 300 python scripts/ln_fwd_perf.py >> gpurun_out/ln_perf.jsonl 2>&1; done
timeout 300 ncu --set full --clock-control none -k regex:"k_ln|k_colred" -c 6 -o gpurun_out/ln_ops_6p2b python scripts/ln_fwd_perf.py > gpurun_out/ncu_ln.log 2>&1
timeout 600 python bench.py --second-config none --no-profile-p8 --no-cpu-baseline --no-e2e > gpurun_out/bench_ln.log 2>&1; echo "rc $?" >> gpurun_out/bench_ln.log
tail -3 gpurun_out/t3.log; cat gpurun_out/ln_perf.jsonl; tail -c 300 gpurun_out/bench_ln.log
