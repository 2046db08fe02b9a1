set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kl.py tests/test_gpu_shifts.py -q -x > gpurun_out/ab10_tests.log 2>&1; tail -2 gpurun_out/ab10_tests.log
ENCF_KS_TMA_T=128 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "rotations or keyswitch or tensor" > gpurun_out/ab10_tests128.log 2>&1; tail -2 gpurun_out/ab10_tests128.log
for v in base ENCF_KS_TMA_T=128; do
  envs=$v; [ "$v" = base ] && envs=""
  env $envs timeout 600 python bench.py --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/ab10_bench_$v.json
  python - gpurun_out/ab10_bench_$v.json "$v" <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); k=d['kernel_time_ms_per_step']
print(sys.argv[2], d['value'], 'ntt', k.get('ntt'), 'mac', k.get('diag_mac'), 'frac', d['roofline_hbm']['frac'], 'ks_inner', k.get('ks_inner'), 'ks_psi', k.get('ks_psi'), d['phase_ms'])
PY
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:diag_mac_tma --launch-skip 0 --launch-count 2 \
    -o gpurun_out/ab10_ncu_diag_mac python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo "ncu mac rc=$?"
