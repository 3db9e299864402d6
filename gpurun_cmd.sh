timeout 900 python scripts/torch_bf16_baseline_error.py 6.2B > gpurun_out/torch62.log 2>&1; tail -5 gpurun_out/torch62.log
timeout 900 python scripts/torch_bf16_baseline_error.py 1.5B > gpurun_out/torch15.log 2>&1; tail -5 gpurun_out/torch15.log
timeout 600 python scripts/elementwise_qkv.py 1.5B > gpurun_out/qkv15.json 2> gpurun_out/qkv15.err; tail -3 gpurun_out/qkv15.err
