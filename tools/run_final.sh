#!/bin/bash
# Round-end evidence (one GPU), part 1: full -m gpu suite + smoke, default bench (e2e + oracle baseline), the other
# workloads, ncu launch list of the timed step, per-phase kernel split.  Outputs: gpurun_out/${TAG}_* (small files).
set -u
mkdir -p gpurun_out
T=${TAG:-fin}
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/${T}_gpu_all.log 2>&1; tail -2 gpurun_out/${T}_gpu_all.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; tail -1 gpurun_out/${T}_smoke.log
timeout 900 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; tail -c 300 gpurun_out/${T}_bench.json; echo
for w in ks gpt2-linear bert-large-layer; do
  timeout 900 python bench.py --workload $w --no-cpu-baseline > gpurun_out/${T}_bench_$w.json 2> gpurun_out/${T}_bench_$w.err; echo "$w rc=$?"
done
timeout 900 python bench.py --ablation wo-scp --no-e2e --no-cpu-baseline > gpurun_out/${T}_bench_wo_scp.json 2> /dev/null; echo "wo-scp rc=$?"
timeout 900 python tools/phase_breakdown.py > gpurun_out/${T}_phase_breakdown.json 2> /dev/null; echo "phases rc=$?"
ENCF_NCU_REGION=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,launch__grid_size --clock-control none \
    --csv --log-file gpurun_out/${T}_launches_full.csv \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo "launches rc=$?"
python tools/step_launches.py gpurun_out/${T}_launches_full.csv > gpurun_out/${T}_launches_step.md
python tools/launch_seq.py gpurun_out/${T}_launches_full.csv --all > gpurun_out/${T}_launches_seq.txt && rm -f gpurun_out/${T}_launches_full.csv
