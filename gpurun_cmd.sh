timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/tests_final.log 2>&1; tail -1 gpurun_out/tests_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
timeout 60 python scripts/attn_perf.py 2>&1 | tail -3 > gpurun_out/attn_perf_r4.jsonl
