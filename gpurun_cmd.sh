mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -q -x -p no:cacheprovider --timeout 900 > gpurun_out/fullsize_tests.log 2>&1; echo "rc $?" >> gpurun_out/fullsize_tests.log
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_gemm -c 14 -o gpurun_out/r02_gemm_6p2b_full python scripts/profile_step.py --config 6.2B --layers 1 --m 2 > gpurun_out/ncu_gemm.log 2>&1
tail -4 gpurun_out/fullsize_tests.log; tail -3 gpurun_out/ncu_gemm.log
