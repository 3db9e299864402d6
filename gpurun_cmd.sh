timeout 900 python bench.py --config 6.2B --no-cpu-baseline > gpurun_out/bench_6p2b.json 2> gpurun_out/bench_6p2b.err; echo rc=$?; tail -2 gpurun_out/bench_6p2b.err
