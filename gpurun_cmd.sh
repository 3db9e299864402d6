mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider > gpurun_out/gputests.log 2>&1; echo "tests rc $?" >> gpurun_out/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/smoke.log
timeout 1500 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc $?" >> gpurun_out/bench.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fwd_tc\|k_bwd_tc -c 2 -o gpurun_out/r02_attn_6p2b_persistent python scripts/attn_one.py 3 1024 32 128 > gpurun_out/ncu_attn.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/r02_launches_6p2b_4layer_m1_final.csv python scripts/profile_step.py --config 6.2B --layers 4 --m 1 > gpurun_out/launch.log 2>&1
tail -3 gpurun_out/gputests.log; tail -2 gpurun_out/smoke.log; head -c 600 gpurun_out/bench.log
