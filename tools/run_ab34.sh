# small-batch NTTs as one fused two-phase launch (ENCF_NTT_FUSED_SMALL = max limb transforms per batch; 0 = off)
set -u
mkdir -p gpurun_out
ENCF_NTT_FUSED_SMALL=36 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kl.py -q -x > gpurun_out/ab34_tests.log 2>&1; tail -1 gpurun_out/ab34_tests.log
for v in 0 12 36 72; do
  ENCF_NTT_FUSED_SMALL=$v timeout 600 python bench.py --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/ab34_bench_$v.json
  python - gpurun_out/ab34_bench_$v.json "$v" <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); k=d['kernel_time_ms_per_step']
print(sys.argv[2], d["value"], {x: k.get(x) for x in ("ntt", "diag_mac", "bconv_batch_kernel")}, d["phase_ms"])
PY
done
mkdir -p /tmp/ncu
timeout 600 ncu --set full --import-source on --clock-control none -k regex:bcast_ntt_kernel --launch-skip 1 --launch-count 1 \
    -o /tmp/ncu/r02s4_bcast_main python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo "ncu bcast rc=$?"
python tools/ncu_table.py /tmp/ncu/r02s4_bcast_main.ncu-rep > gpurun_out/r02s4_ncu_bcast_main.md 2>&1; cat gpurun_out/r02s4_ncu_bcast_main.md
