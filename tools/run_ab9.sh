set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kl.py tests/test_gpu_shifts.py -q -x > gpurun_out/ab9_tests.log 2>&1; tail -3 gpurun_out/ab9_tests.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_fullsize2.py -q -x -k "qkv or ff2 or proj" > gpurun_out/ab9_tests_fs.log 2>&1; tail -3 gpurun_out/ab9_tests_fs.log
for v in base ENCF_MAC_VARIANT=reg; do
  envs=$v; [ "$v" = base ] && envs=""
  env $envs timeout 600 python bench.py --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/ab9_bench_$v.json
  python - gpurun_out/ab9_bench_$v.json "$v" <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); k=d['kernel_time_ms_per_step']
print(sys.argv[2], d['value'], 'ntt', k.get('ntt'), 'mac', k.get('diag_mac'), 'frac', d['roofline_hbm']['frac'], 'bconv', k.get('bconv_batch_kernel'), 'bcast', k.get('bcast_mac'), d['phase_ms'])
PY
done
