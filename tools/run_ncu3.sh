#!/bin/bash
# ncu --set full of single launches inside the timed step (ENCF_NCU_REGION=1 + --profile-from-start off):
# the value kernel's Toeplitz convolution (bcast_ntt_kernel) and a large base conversion (the value Phi-bank
# ModDown, 22nd bconv launch of the step) with the cp.async.bulk input ring (default) and without (BTC_ST=0).
set -u
mkdir -p gpurun_out /tmp/ncu
T=${TAG:-s3}
run() {   # name regex skip [env...]
  local name=$1 rx=$2 skip=$3; shift 3
  env ENCF_NCU_REGION=1 "$@" timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none \
      -k regex:$rx --launch-skip $skip --launch-count 1 -o /tmp/ncu/${T}_$name \
      python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo "ncu $name rc=$?"
}
run bcast_ntt bcast_ntt_kernel 0
run bconv_ring bconv_tc_kernel 21
run bconv_st0 bconv_tc_kernel 21 ENCF_LIB_OVERRIDE=build_variants/lib_st0.so
python tools/ncu_table.py /tmp/ncu/${T}_*.ncu-rep > gpurun_out/${T}_ncu_table.md 2>&1
for f in /tmp/ncu/${T}_*.ncu-rep; do
  b=$(basename $f .ncu-rep)
  ncu -i $f --page raw --csv > gpurun_out/${b}_raw.csv 2>/dev/null
  ncu -i $f --page details --csv > gpurun_out/${b}_details.csv 2>/dev/null
done
gzip -f gpurun_out/${T}_*_raw.csv gpurun_out/${T}_*_details.csv
cat gpurun_out/${T}_ncu_table.md
