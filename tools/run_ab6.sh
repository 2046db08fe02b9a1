set -u
mkdir -p gpurun_out
for v in smtw nosmtw; do
  lib=""; [ $v = nosmtw ] && lib="ENCF_LIB_OVERRIDE=build_variants/libencf_nosmtw.so"
  env $lib timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none -k regex:ntt_ --csv \
      --log-file gpurun_out/ab6_ntt_$v.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
  echo "$v ncu rc=$?"
  env $lib python bench.py --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['value'], d['kernel_time_ms_per_step']['ntt'])"
done
