#!/bin/bash
# Baseline GPU pass for a session: full -m gpu suite, default bench, ncu launch list of the timed step.
set -u
mkdir -p gpurun_out
T=${TAG:-s2}
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/${T}_gpu_all.log 2>&1; tail -2 gpurun_out/${T}_gpu_all.log
timeout 900 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; tail -c 3000 gpurun_out/${T}_bench.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${T}_ncu_bench.log 2>&1
echo "ncu rc=$?"
