set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kl.py -q -x > gpurun_out/r2_t6_kl.log 2>&1; tail -2 gpurun_out/r2_t6_kl.log
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/r2_t6_all.log 2>&1; tail -2 gpurun_out/r2_t6_all.log
timeout 600 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/r2_bench3.json 2> gpurun_out/r2_bench3.err
ENCF_MAC_LEGACY=1 timeout 600 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/r2_bench3_legacymac.json 2>&1
for f in gpurun_out/r2_bench3*.json; do python - "$f" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], d['value'], d['kernel_time_ms_per_step'].get('ntt'), d['kernel_time_ms_per_step'].get('diag_mac'), d['roofline_hbm']['frac'], d['phase_ms'])
except Exception as e: print(sys.argv[1], 'ERR', e)
PY
done
