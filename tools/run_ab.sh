#!/bin/bash
# A/B pass: fast parity subset, then bench variants selected by environment switches (TAG, VARIANTS).
set -u
mkdir -p gpurun_out
T=${TAG:-ab}
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kl.py tests/test_gpu_shifts.py tests/test_gpu_graph.py -q -x > gpurun_out/${T}_tests.log 2>&1; tail -2 gpurun_out/${T}_tests.log
for v in ${VARIANTS:-"base"}; do
  envs=$(echo "$v" | tr '+' ' '); [ "$v" = base ] && envs=""
  env $envs timeout 600 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/${T}_bench_${v}.json 2> gpurun_out/${T}_bench_${v}.err
  python - "gpurun_out/${T}_bench_${v}.json" "$v" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); k=d['kernel_time_ms_per_step']
    print(sys.argv[2], d['value'], 'ntt', k.get('ntt'), 'mac', k.get('diag_mac'), 'bconv', k.get('bconv_batch_kernel'), 'ks_inner', k.get('ks_inner'), d['phase_ms'])
except Exception as e: print(sys.argv[2], 'ERR', e)
PY
done
