timeout 2000 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -rf 2>&1 | grep -E "Error|FAILED|passed|failed" | tail -30 > gpurun_out/gpu_tests.log
tail -30 gpurun_out/gpu_tests.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-profile-p8 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 1500 gpurun_out/bench.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1])
for dd in (d, d.get('second_config')):
    if not dd: continue
    r=dd['roofline']
    print(dd['config']['model'], dd['value'], dd['ms_per_step'], r['frac'], {k:(round(v['ms_total'],1), round(v['tflops'])) for k,v in r['per_class'].items()}, {k:v.get('ms_total') for k,v in r['hbm_kernels']['classes'].items()}, r['unaccounted_ms_per_step'], dd['gpu_launches'])
PY
