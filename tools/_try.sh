# quick check of a solve-kernel change: bitwise fingerprints, phase timers, solver tests, bench
mkdir -p gpurun_out
timeout 600 python tools/bitcheck.py gpurun_out/bitcheck_new.json > gpurun_out/bitcheck.log 2>&1; echo "bitcheck rc=$?"
python - <<'PY'
import json
a=json.load(open('profiles/r02/bitcheck_6e5fece.json')); b=json.load(open('gpurun_out/bitcheck_new.json'))
for k in a: print(k, 'SAME' if a[k]==b.get(k) else ('DIFF', a[k]['its'], b.get(k,{}).get('its')))
PY
timeout 300 python tools/phase_seq.py 2>&1 | grep phase_timers | cut -c1-420
timeout 900 python -m pytest tests/test_gpu_solvers.py tests/test_gpu_pipeline.py tests/test_gpu_gpc.py -x -q -m gpu 2>&1 | tail -3
timeout 600 python bench.py > gpurun_out/bench_try.jsonl 2> gpurun_out/bench_try.err; echo "bench rc=$?"
python - <<'PY'
import json
j=json.loads(open('gpurun_out/bench_try.jsonl').read().strip().splitlines()[-1])
print('value', j['value'], 'ms', j['ms_per_step'], 'frac', j['roofline']['frac'], 'e2e', j['e2e']['value'], 'cg_ms', j['plain_cg']['sequence_ms'], 'c3', j.get('config3_single_gpu',{}).get('sequence_ms'), j.get('config3_single_gpu',{}).get('solve_kernel_roofline',{}).get('frac'))
PY
