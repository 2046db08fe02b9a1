set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kl.py tests/test_gpu_shifts.py tests/test_gpu_graph.py -q -x > gpurun_out/ab14_tests.log 2>&1; tail -2 gpurun_out/ab14_tests.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k "score or value" > gpurun_out/ab14_tests_fs.log 2>&1; tail -2 gpurun_out/ab14_tests_fs.log
timeout 600 python bench.py --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/ab14_bench.json
python - gpurun_out/ab14_bench.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); k=d['kernel_time_ms_per_step']
print(d['value'], 'ntt', k.get('ntt'), 'mac', k.get('diag_mac'), 'ks_inner', k.get('ks_inner'), 'ks_psi', k.get('ks_psi'), 'bconv', k.get('bconv_batch_kernel'), 'bcast', k.get('bcast_mac'), d['phase_ms'])
PY
