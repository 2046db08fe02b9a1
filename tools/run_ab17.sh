set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kl.py tests/test_gpu_shifts.py tests/test_gpu_graph.py -q -x > gpurun_out/ab17_tests.log 2>&1; tail -2 gpurun_out/ab17_tests.log
timeout 900 python bench.py --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/ab17_bench.json
ENCF_MODUP_NTT_GATHER=1 timeout 900 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/ab17_bench_large.json
for f in gpurun_out/ab17_bench.json gpurun_out/ab17_bench_large.json; do python - $f <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); k=d['kernel_time_ms_per_step']
print(sys.argv[1], d['value'], 'e2e', d['e2e']['value'], 'ntt', k.get('ntt'), 'mac', k.get('diag_mac'), 'bcast', k.get('bcast_mac'), d['phase_ms'])
PY
done
