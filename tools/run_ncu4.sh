#!/bin/bash
# Round-end ncu --set full of the top kernels (one launch each, cold and serialised under ncu); only the summary table and
# the gzipped raw/details pages come back.  TAG from the environment.
set -u
mkdir -p gpurun_out /tmp/ncu
T=${TAG:-fin}
cap() {   # name regex skip
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$2 --launch-skip $3 --launch-count 1 \
      -o /tmp/ncu/${T}_$1 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo "ncu $1 rc=$?"
}
cap diag_mac diag_mac_tma_kernel 1
cap bconv bconv_tc_kernel 2
cap ks_inner ks_inner_tma_kernel 2
cap ks_group ks_group_tma_kernel 0
cap bcast_ntt bcast_ntt_kernel 0
cap ks_psi ks_psi_tma_kernel 0
cap tensor tensor_csr_kernel 0
timeout 600 ncu --set full --import-source on --clock-control none -k regex:ntt_ --launch-skip 8 --launch-count 4 \
    -o /tmp/ncu/${T}_ntt python tools/ntt_bench.py > /dev/null 2>&1; echo "ncu ntt rc=$?"
python tools/ncu_table.py /tmp/ncu/${T}_*.ncu-rep > gpurun_out/${T}_ncu_table.md 2>&1
for f in /tmp/ncu/${T}_*.ncu-rep; do
  b=$(basename $f .ncu-rep)
  ncu -i $f --page raw --csv > gpurun_out/${b}_raw.csv 2>/dev/null
done
gzip -f gpurun_out/${T}_*_raw.csv
cat gpurun_out/${T}_ncu_table.md
