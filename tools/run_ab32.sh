# narrow-limb plaintext MAC: warps 4-7 on the FP64 pipe (default) vs integer pipe only (ENCF_MAC_FP=0)
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kl.py tests/test_gpu_shifts.py tests/test_gpu_fullsize.py tests/test_gpu_fullsize2.py -q -x > gpurun_out/ab32_tests.log 2>&1; tail -2 gpurun_out/ab32_tests.log
for v in base ENCF_MAC_FP=0; do
  envs=$v; [ "$v" = base ] && envs=""
  env $envs timeout 600 python bench.py --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/ab32_bench_$v.json
  python - gpurun_out/ab32_bench_$v.json "$v" <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); k=d['kernel_time_ms_per_step']
print(sys.argv[2], d["value"], {x: k.get(x) for x in ("ntt", "diag_mac", "bconv_batch_kernel")}, d.get("roofline_hbm", {}).get("frac"), d["phase_ms"])
PY
done
