# fused P sigma_g(c0) lift in the key-switch inner product (rotations kept in Q_L u P): parity + bench
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kl.py tests/test_gpu_shifts.py tests/test_gpu_fullsize.py tests/test_gpu_graph.py -q -x > gpurun_out/ab27_tests.log 2>&1; tail -2 gpurun_out/ab27_tests.log
ENCF_KS_TMA=0 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "projection or rotations or value or score" > gpurun_out/ab27_tests_kstma0.log 2>&1; tail -1 gpurun_out/ab27_tests_kstma0.log
timeout 600 python bench.py --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/ab27_bench.json
python - gpurun_out/ab27_bench.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); k=d['kernel_time_ms_per_step']
print(d["value"], {x: k.get(x) for x in ("ntt", "ks_inner", "gather_copy_kernel", "lift_add_kernel", "bcast_mac")}, d["phase_ms"])
PY
