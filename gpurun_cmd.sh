mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
# 1. launch list of one 6.2B microbatch (4 layers + head + optimizer)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/r02_launches_6p2b_4layer_m1.csv python scripts/profile_step.py --config 6.2B --layers 4 --m 1 > gpurun_out/launch.log 2>&1
# 2. GEMM DRAM bytes (2 layers + head)
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --profile-from-start off -k regex:k_gemm --csv --log-file gpurun_out/r02_gemm_dram_6p2b_2layer_m1.csv python scripts/profile_step.py --config 6.2B --layers 2 --m 1 > gpurun_out/dram.log 2>&1
# 3. sustained GEMM vs cuBLAS at the 6.2B shapes
timeout 600 python scripts/gemm_sustained.py --model 6.2B --secs 1.5 > gpurun_out/r02_gemm_sustained_6p2b.jsonl 2>&1
# 4. attention perf at both shapes
timeout 300 python scripts/attn_perf.py > gpurun_out/r02_attn_perf.jsonl 2>&1
# 5. full ncu of the attention kernels at the 6.2B shape
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fwd_tc\|k_bwd_tc -c 2 -o gpurun_out/r02_attn_6p2b python scripts/attn_one.py 3 1024 32 128 > gpurun_out/ncu_attn.log 2>&1
tail -3 gpurun_out/*.log; cat gpurun_out/r02_gemm_sustained_6p2b.jsonl gpurun_out/r02_attn_perf.jsonl
