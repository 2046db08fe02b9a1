#!/bin/bash
# compute-sanitizer runs on the small-parameter (P12 / P13) GPU parity tests; logs under gpurun_out/.
# usage (on the GPU box): bash tools/sanitize.sh
set -u
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
SEL="projection_config1 or rotations_conj or tensor_relin or score_and_export or value_bit_exact or export_c2m or rotfirst or psi_bit or restricted or phase_alignment or unit_partials"
timeout 1500 $CS --tool memcheck --target-processes all --print-limit 50 --error-exitcode 9 \
    python -m pytest tests/test_gpu_parity.py tests/test_gpu_shifts.py -q -k "$SEL" > gpurun_out/sanitizer_memcheck.log 2>&1
echo "memcheck rc=$?" >> gpurun_out/sanitizer_memcheck.log
timeout 1500 $CS --tool racecheck --racecheck-report hazard --target-processes all --print-limit 50 --error-exitcode 9 \
    python -m pytest tests/test_gpu_parity.py tests/test_gpu_shifts.py -q -k "projection_config1 or rotations_conj_bit_exact[8] or value_bit_exact or rotfirst_bit_exact" > gpurun_out/sanitizer_racecheck.log 2>&1
echo "racecheck rc=$?" >> gpurun_out/sanitizer_racecheck.log
timeout 900 $CS --tool synccheck --target-processes all --print-limit 50 --error-exitcode 9 \
    python -m pytest tests/test_gpu_parity.py -q -k "projection_config1 or score_and_export" > gpurun_out/sanitizer_synccheck.log 2>&1
echo "synccheck rc=$?" >> gpurun_out/sanitizer_synccheck.log
for f in gpurun_out/sanitizer_*.log; do tail -n 3 "$f"; done
