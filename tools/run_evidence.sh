#!/bin/bash
# Round evidence pass (one GPU): full -m gpu suite, default bench (e2e + oracle baseline), ncu launch list of the
# timed step, ncu --set full of the top kernels.  Outputs: gpurun_out/${TAG}_*.
set -u
mkdir -p gpurun_out
T=${TAG:-ev}
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/${T}_gpu_all.log 2>&1; tail -2 gpurun_out/${T}_gpu_all.log
timeout 900 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; tail -c 400 gpurun_out/${T}_bench.json; echo
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo "launches rc=$?"
for k in diag_mac_tma_kernel bconv_tc_kernel ks_inner_tma_kernel bcast_mac_kernel ks_psi_kernel; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k --launch-skip 2 --launch-count 1 \
      -o gpurun_out/${T}_ncu_$k python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo "ncu $k rc=$?"
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:ntt_ --launch-skip 8 --launch-count 4 \
    -o gpurun_out/${T}_ncu_ntt python tools/ntt_bench.py > /dev/null 2>&1; echo "ncu ntt rc=$?"
