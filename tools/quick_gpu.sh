# quick GPU iteration: parity tests of the Mode U split paths + a short bench (no e2e/configs/cpu)
set -x
mkdir -p gpurun_out
T=${TESTS:-tests/test_gpu_parity.py tests/test_gpu_timed_configs.py tests/test_gpu_fullsize.py}
timeout 900 python -m pytest $T -x -q > gpurun_out/quick_pytest.log 2>&1; tail -5 gpurun_out/quick_pytest.log
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-unfused --no-configs --e2e-steps 2 > gpurun_out/quick_bench.json 2> gpurun_out/quick_bench.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/quick_bench.json').read().strip().splitlines()[-1])
print('value', d['value'], 'ms', d['ms_per_step'], 'parity', d['parity']['mismatches'], 'e2e', d['e2e']['value'])
r=d['roofline']; print('scan frac', r['frac'], 'stage', r['stage_upsample_nms'])
for k,v in d['stages'].items():
    if 'ms_per_launch' in v: print(k, round(v['ms_per_launch'],4))
PY
tail -3 gpurun_out/quick_bench.err
