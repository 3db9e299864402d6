mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
for h in 0 1 2 3; do
  echo "# ZB_GEMM_CHINT=$h" >> gpurun_out/r02_gemm_chint.jsonl
  ZB_GEMM_CHINT=$h timeout 600 python scripts/gemm_sustained.py --model 6.2B --secs 1.0 >> gpurun_out/r02_gemm_chint.jsonl 2>&1
done
for h in 0 3; do
  ZB_GEMM_CHINT=$h timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --profile-from-start off -k regex:k_gemm --csv --log-file gpurun_out/r02_gemm_dram_chint$h.csv python scripts/profile_step.py --config 6.2B --layers 2 --m 2 > /dev/null 2>&1
done
cat gpurun_out/r02_gemm_chint.jsonl
