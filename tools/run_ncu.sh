#!/bin/bash
# Round-end evidence, part 2: ncu --set full of the top kernels; only the summary tables come back (the .ncu-rep
# files exceed gpurun's 64 MiB return limit).  KERNELS / TAG from the environment.
set -u
mkdir -p gpurun_out /tmp/ncu
T=${TAG:-fin}
for k in ${KERNELS:-diag_mac_tma_kernel bconv_tc_kernel ks_inner_tma_kernel bcast_mac_kernel ks_psi_tma_kernel ks_rotsum_kernel}; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k --launch-skip 2 --launch-count 1 \
      -o /tmp/ncu/${T}_$k python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo "ncu $k rc=$?"
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:ntt_ --launch-skip 8 --launch-count 4 \
    -o /tmp/ncu/${T}_ntt python tools/ntt_bench.py > /dev/null 2>&1; echo "ncu ntt rc=$?"
python tools/ncu_table.py /tmp/ncu/${T}_*.ncu-rep > gpurun_out/${T}_ncu_table.md 2>&1
for f in /tmp/ncu/${T}_*.ncu-rep; do
  b=$(basename $f .ncu-rep)
  ncu -i $f --page raw --csv > gpurun_out/${b}_raw.csv 2>/dev/null
  ncu -i $f --page details --csv > gpurun_out/${b}_details.csv 2>/dev/null
done
gzip -f gpurun_out/${T}_*_raw.csv gpurun_out/${T}_*_details.csv
du -sh gpurun_out
