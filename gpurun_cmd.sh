timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/tests_final.log 2>&1; tail -1 gpurun_out/tests_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_22l.csv python scripts/profile_step.py --layers 22 --m 1 > gpurun_out/launches.log 2>&1; echo ncu rc=$?
