#!/bin/bash
# build NTT variants on the GPU box and time each (kernel experiments): us per limb transform, FP64 / integer path
set -e
mkdir -p /tmp/var gpurun_out
for v in "NTT_MINB=3" "NTT_MINB=4" "NTT_MINB=5" "NTT_MINB=6"; do
  python -c "import sys; sys.path.insert(0,'.'); from paper_2604_09975_b200 import build as b; b.build_variant('/tmp/var/lib_$v.so', ['$v'])" > /dev/null 2>&1
  echo "$v fp64 $(ENCF_LIB_OVERRIDE=/tmp/var/lib_$v.so python tools/ntt_bench.py) int $(ENCF_NTT_INT_ONLY=1 ENCF_LIB_OVERRIDE=/tmp/var/lib_$v.so python tools/ntt_bench.py)"
done
