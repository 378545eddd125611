timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -4
timeout 300 python scripts/e2e_breakdown.py 2>&1 | head -1
timeout 600 python bench.py --no-throughput > gpurun_out/bench_e2e.json 2> gpurun_out/bench_e2e.err; echo bench rc=$?
python - <<'P'
import json; d=json.loads(open('gpurun_out/bench_e2e.json').read().strip().splitlines()[-1])
print('value', d['value'], 'ms', d['ms_per_step'], 'e2e', d['e2e']['value'], d['e2e']['s_per_call'], 'grad', d['gradient']['s_per_iter'])
P
