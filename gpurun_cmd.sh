mkdir -p gpurun_out
rm -f gpurun_out/delta_perf2.jsonl
for v in new old new old; do echo "# delta $v" >> gpurun_out/delta_perf2.jsonl; if [ $v = old ]; then export ZB_DELTA_OLD=1; else unset ZB_DELTA_OLD; fi; timeout 300 python scripts/attn_perf.py >> gpurun_out/delta_perf2.jsonl 2>&1; done
cat gpurun_out/delta_perf2.jsonl
