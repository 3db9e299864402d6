mkdir -p gpurun_out
ZB_GEMM_CHINT=8 timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_wgroup.py -q -x -p no:cacheprovider > gpurun_out/la_tests.log 2>&1; echo "rc $?" >> gpurun_out/la_tests.log
for h in 0 8 0 8; do echo "# CHINT $h" >> gpurun_out/w_loadadd.jsonl; ZB_GEMM_CHINT=$h timeout 600 python scripts/gemm_w_c3.py --secs 1.0 >> gpurun_out/w_loadadd.jsonl 2>&1; done
tail -3 gpurun_out/la_tests.log; cat gpurun_out/w_loadadd.jsonl
