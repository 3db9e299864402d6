mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
timeout 600 python -m pytest tests/test_gpu_attention.py -q -x -p no:cacheprovider > gpurun_out/attn_tests.log 2>&1; echo "rc $?" >> gpurun_out/attn_tests.log
timeout 300 python scripts/attn_perf.py > gpurun_out/r02_attn_perf_grid1d.jsonl 2>&1
timeout 900 python scripts/gemm_w_c3.py --secs 1.0 > gpurun_out/r02_gemm_w_c3_variants.jsonl 2>&1
S=gpurun_out/r02_sanitizer_race.txt
echo "# compute-sanitizer racecheck, round 2 (B200)" > $S
run() { echo "## $1 $2 [-k $3]" >> $S; timeout 900 compute-sanitizer --tool $1 --print-limit 20 python -m pytest $2 -k "$3" -q -x -p no:cacheprovider --timeout 800 2>&1 | grep -v "^$" | tail -8 >> $S; }
run racecheck tests/test_gpu_attention.py "b2s256a3d64 and bf16"
run racecheck tests/test_gpu_attention.py "b1s256a2d128 and bf16"
run racecheck tests/test_gpu_attention.py "b2s192a2d96 and bf16"
run racecheck tests/test_gpu_gemm.py "1024x192x64 and bf16"
run racecheck tests/test_gpu_gemm.py "512x512x4096 and bf16"
run racecheck tests/test_gpu_gemm.py "512x640x256 and bf16"
cat gpurun_out/attn_tests.log | tail -3; cat gpurun_out/r02_attn_perf_grid1d.jsonl gpurun_out/r02_gemm_w_c3_variants.jsonl; cat $S
