mkdir -p gpurun_out
md5sum paper_2401_10241_b200/libzb.so > gpurun_out/final4_md5.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/final4_gpu_tests.log 2>&1; echo "rc $?" >> gpurun_out/final4_gpu_tests.log
timeout 900 python bench.py > gpurun_out/final4_bench.log 2>&1; echo "rc $?" >> gpurun_out/final4_bench.log
tail -3 gpurun_out/final4_gpu_tests.log; tail -c 300 gpurun_out/final4_bench.log
