set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_graph.py -q -x > gpurun_out/ab18_tests.log 2>&1; tail -2 gpurun_out/ab18_tests.log
for r in 1 2 3; do
  timeout 900 python bench.py --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/ab18_bench_$r.json
  python - gpurun_out/ab18_bench_$r.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); k=d['kernel_time_ms_per_step']
print(d['value'], 'e2e', d['e2e']['value'], d['e2e'].get('clocks'), 'dev clocks', d['clocks'], 'ntt', k.get('ntt'))
PY
done
