mkdir -p gpurun_out
timeout 900 python bench.py --second-config none --no-profile-p8 --no-cpu-baseline > gpurun_out/c34_bench.log 2>&1; echo "rc $?" >> gpurun_out/c34_bench.log
tail -c 400 gpurun_out/c34_bench.log
