mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
timeout 1200 python -m pytest tests/test_gpu_dp_shim.py tests/test_gpu_nccl_shim.py -q -x --timeout 900 -p no:cacheprovider > gpurun_out/dp.log 2>&1; echo "rc $?" >> gpurun_out/dp.log
S=gpurun_out/r02_sanitizer.txt
echo "# compute-sanitizer, round 2 (B200)" > $S
run() { echo "## $1 $2" >> $S; timeout 900 compute-sanitizer --tool $1 --print-limit 20 python -m pytest $2 -q -x -p no:cacheprovider --timeout 800 2>&1 | grep -v "^$" | tail -8 >> $S; }
run racecheck "tests/test_gpu_attention.py -k bf16-b2s256a3d64"
run racecheck "tests/test_gpu_attention.py -k bf16-b1s256a2d128"
run racecheck "tests/test_gpu_gemm.py -k bf16-1024x192"
run racecheck "tests/test_gpu_gemm.py -k bf16-512x512x4096"
run memcheck "tests/test_gpu_ops.py"
run memcheck "tests/test_gpu_pipeline_loopback.py -k clean"
run synccheck "tests/test_gpu_gemm.py -k bf16"
run memcheck "tests/test_gpu_wgroup.py"
tail -5 gpurun_out/dp.log; cat $S
