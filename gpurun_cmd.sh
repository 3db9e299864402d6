mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/final_gpu_tests.log 2>&1; echo "rc $?" >> gpurun_out/final_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final_smoke.log 2>&1; echo "rc $?" >> gpurun_out/final_smoke.log
timeout 900 python bench.py > gpurun_out/final_bench.log 2>&1; echo "rc $?" >> gpurun_out/final_bench.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/final_ref.log 2>&1; echo "rc $?" >> gpurun_out/final_ref.log
tail -3 gpurun_out/final_gpu_tests.log; tail -2 gpurun_out/final_smoke.log; tail -c 400 gpurun_out/final_bench.log; tail -c 400 gpurun_out/final_ref.log
