# fused P d0, P d1 relinearisation lifts + grouped giant-step sums in the projection (ENCF_PROJ_GROUP=0: previous path)
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kl.py tests/test_gpu_shifts.py tests/test_gpu_fullsize.py tests/test_gpu_graph.py tests/test_gpu_sharded.py -q -x > gpurun_out/ab28_tests.log 2>&1; tail -2 gpurun_out/ab28_tests.log
ENCF_KS_TMA=0 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "projection or rotations or value or score or relin" > gpurun_out/ab28_tests_kstma0.log 2>&1; tail -1 gpurun_out/ab28_tests_kstma0.log
ENCF_PROJ_GROUP=0 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shifts.py -q -x -k "projection or unit" > gpurun_out/ab28_tests_pg0.log 2>&1; tail -1 gpurun_out/ab28_tests_pg0.log
for v in base ENCF_PROJ_GROUP=0; do
  envs=$v; [ "$v" = base ] && envs=""
  env $envs timeout 600 python bench.py --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/ab28_bench_$v.json
  python - gpurun_out/ab28_bench_$v.json "$v" <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); k=d['kernel_time_ms_per_step']
print(sys.argv[2], d["value"], {x: k.get(x) for x in ("ntt", "ks_inner", "gather_copy_kernel", "sum_csr_kernel", "bcast_mac")}, d["phase_ms"])
PY
done
