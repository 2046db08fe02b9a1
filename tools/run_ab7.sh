set -u
mkdir -p gpurun_out
echo "smtw fp64 $(python tools/ntt_bench.py) int $(ENCF_NTT_INT_ONLY=1 python tools/ntt_bench.py)"
echo "ldg  fp64 $(ENCF_LIB_OVERRIDE=build_variants/libencf_nosmtw.so python tools/ntt_bench.py) int $(ENCF_LIB_OVERRIDE=build_variants/libencf_nosmtw.so ENCF_NTT_INT_ONLY=1 python tools/ntt_bench.py)"
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kl.py tests/test_gpu_shifts.py -q -x > gpurun_out/ab7_tests.log 2>&1; tail -3 gpurun_out/ab7_tests.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k "value" > gpurun_out/ab7_tests_fs.log 2>&1; tail -3 gpurun_out/ab7_tests_fs.log
for v in base ENCF_LIB_OVERRIDE=build_variants/libencf_nosmtw.so; do
  envs=$v; [ "$v" = base ] && envs=""
  env $envs timeout 600 python bench.py --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/ab7_bench.json
  python - gpurun_out/ab7_bench.json "$v" <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); k=d['kernel_time_ms_per_step']
print(sys.argv[2][-20:], d['value'], 'ntt', k.get('ntt'), 'mac', k.get('diag_mac'), 'bconv', k.get('bconv_batch_kernel'), 'bcast', k.get('bcast_mac'), d['phase_ms'])
PY
done
