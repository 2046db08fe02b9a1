set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_graph.py tests/test_gpu_kl.py -q -x > gpurun_out/ab20_tests.log 2>&1; tail -2 gpurun_out/ab20_tests.log
for v in base ENCF_KS_SERIAL=1; do
  envs=$v; [ "$v" = base ] && envs=""
  env $envs timeout 600 python bench.py --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/ab20_bench_$v.json
  python - gpurun_out/ab20_bench_$v.json "$v" <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); k=d['kernel_time_ms_per_step']
print(sys.argv[2], d['value'], 'ntt', k.get('ntt'), d['phase_ms'])
PY
done
