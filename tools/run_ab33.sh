# BConv persistent grid: 4 (default) vs 5 vs 6 CTAs per SM (occupancy-capped)
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kl.py -q -x > gpurun_out/ab33_tests.log 2>&1; tail -2 gpurun_out/ab33_tests.log
for v in base ps5 ps6; do
  lib=""; [ "$v" != base ] && lib="ENCF_LIB_OVERRIDE=build_variants/lib_$v.so"
  env $lib timeout 600 python bench.py --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/ab33_bench_$v.json
  python - gpurun_out/ab33_bench_$v.json "$v" <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); k=d['kernel_time_ms_per_step']
print(sys.argv[2], d["value"], {x: k.get(x) for x in ("ntt", "bconv_batch_kernel", "diag_mac", "ks_inner")}, d["phase_ms"])
PY
done
