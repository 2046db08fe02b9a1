# batched complexify in the bench step (encf_complexify_many)
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_graph.py -q -x > gpurun_out/ab37_tests.log 2>&1; tail -1 gpurun_out/ab37_tests.log
for i in 1 2; do
  timeout 600 python bench.py --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/ab37_bench_$i.json
  python - gpurun_out/ab37_bench_$i.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); k=d['kernel_time_ms_per_step']
print(d["value"], {x: k.get(x) for x in ("ntt", "rescale_prep_batch_kernel", "bcast_mac")}, d["phase_ms"])
PY
done
