# A/B: value Toeplitz kernel, persistent with cp.async.bulk-staged windows (default) vs direct loads
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kl.py tests/test_gpu_shifts.py tests/test_gpu_fullsize.py -q -x > gpurun_out/ab25_tests.log 2>&1; tail -2 gpurun_out/ab25_tests.log
for v in base ENCF_BCAST_NOTMA=1; do
  lib=$v; [ "$v" = base ] && lib=""
  env $lib timeout 600 python bench.py --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/ab25_bench_$v.json
  python - gpurun_out/ab25_bench_$v.json "$v" <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); k=d['kernel_time_ms_per_step']
print(sys.argv[2], d['value'], 'ntt', k.get('ntt'), 'bconv', k.get('bconv_batch_kernel'), 'bcast', k.get('bcast_mac'), d['phase_ms'])
PY
done
