# A/B: integer-NTT q = 2^60 - c Shoup remainder (NTT_CQ) and the value Toeplitz kernel's occupancy (TZ_MINB)
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kl.py -q -x > gpurun_out/ab21_tests.log 2>&1; tail -2 gpurun_out/ab21_tests.log
for v in base cq0 tz4; do
  lib=""; [ "$v" != base ] && lib="ENCF_LIB_OVERRIDE=build_variants/lib_$v.so"
  echo "$v ntt(fp64,int) $(env $lib python tools/ntt_bench.py) $(env $lib ENCF_NTT_INT_ONLY=1 python tools/ntt_bench.py)"
  env $lib timeout 600 python bench.py --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/ab21_bench_$v.json
  python - gpurun_out/ab21_bench_$v.json "$v" <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); k=d['kernel_time_ms_per_step']
print(sys.argv[2], d['value'], 'ntt', k.get('ntt'), 'bcast', k.get('bcast_mac'), d['phase_ms'])
PY
done
