set -u
mkdir -p gpurun_out
for n in 1 2 4 6; do echo "ctas/SM=$n"; TC_CTAS_PER_SM=$n ./tools/micro/bconv_tc; done > gpurun_out/ab4_bconv_tc.txt 2>&1; cat gpurun_out/ab4_bconv_tc.txt
echo "fp64 $(python tools/ntt_bench.py) int $(ENCF_NTT_INT_ONLY=1 python tools/ntt_bench.py)"
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kl.py tests/test_gpu_shifts.py -q -x > gpurun_out/ab4_tests.log 2>&1; tail -2 gpurun_out/ab4_tests.log
timeout 600 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/ab4_bench.json 2> gpurun_out/ab4_bench.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/ab4_bench.json').read().strip().splitlines()[-1]); k=d['kernel_time_ms_per_step']
print(d['value'], 'ntt', k.get('ntt'), 'mac', k.get('diag_mac'), 'bconv', k.get('bconv_batch_kernel'), 'ks_inner', k.get('ks_inner'), d['phase_ms'])
PY
timeout 600 ncu --set full -k regex:ntt_rows --launch-skip 4 --launch-count 1 -o gpurun_out/ab4_ntt_rows python tools/ntt_bench.py > /dev/null 2>&1; echo ncu $?
