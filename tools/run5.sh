set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shifts.py tests/test_gpu_graph.py tests/test_gpu_sharded.py -q -x > gpurun_out/r2_t5.log 2>&1
tail -2 gpurun_out/r2_t5.log
timeout 900 python bench.py > gpurun_out/r2_bench2.json 2> gpurun_out/r2_bench2.err
ENCF_MAC_LEGACY=1 timeout 600 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/r2_bench2_legacymac.json 2>&1
ENCF_NTT_CHUNK_MB=0 timeout 600 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/r2_bench2_nochunk.json 2>&1
ENCF_NTT_CHUNK_MB=64 timeout 600 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/r2_bench2_chunk64.json 2>&1
for f in gpurun_out/r2_bench2*.json; do python - "$f" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], d['value'], d['kernel_time_ms_per_step'].get('ntt'), d['kernel_time_ms_per_step'].get('diag_mac'), d['roofline_hbm']['frac'])
except Exception as e: print(sys.argv[1], 'ERR', e)
PY
done
