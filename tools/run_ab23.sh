# A/B: base-conversion epilogue, one TMEM load per output (BTC_LD4=0) vs one x32 load per four outputs
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kl.py -q -x > gpurun_out/ab23_tests.log 2>&1; tail -2 gpurun_out/ab23_tests.log
for v in base ld1; do
  lib=""; [ "$v" != base ] && lib="ENCF_LIB_OVERRIDE=build_variants/lib_$v.so"
  env $lib timeout 600 python bench.py --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/ab23_bench_$v.json
  python - gpurun_out/ab23_bench_$v.json "$v" <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); k=d['kernel_time_ms_per_step']
print(sys.argv[2], d['value'], 'ntt', k.get('ntt'), 'bconv', k.get('bconv_batch_kernel'), 'bcast', k.get('bcast_mac'), d['phase_ms'])
PY
done
