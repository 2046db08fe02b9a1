set -u
mkdir -p gpurun_out
echo "fp64 $(python tools/ntt_bench.py) int $(ENCF_NTT_INT_ONLY=1 python tools/ntt_bench.py)"
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kl.py tests/test_gpu_shifts.py tests/test_gpu_graph.py -q -x > gpurun_out/ab5_tests.log 2>&1; tail -3 gpurun_out/ab5_tests.log
for v in base ENCF_BCONV_TC=0; do
  envs=$v; [ "$v" = base ] && envs=""
  env $envs timeout 600 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/ab5_bench_$v.json 2> gpurun_out/ab5_bench_$v.err
  python - gpurun_out/ab5_bench_$v.json $v <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); k=d['kernel_time_ms_per_step']
print(sys.argv[2], d['value'], 'ntt', k.get('ntt'), 'mac', k.get('diag_mac'), 'bconv', k.get('bconv_batch_kernel'), 'ks_inner', k.get('ks_inner'), d['phase_ms'])
PY
done
