set -u
mkdir -p gpurun_out
./tools/micro/bconv_tc > gpurun_out/ab3_bconv_tc.txt 2>&1; echo "bconv_tc rc=$?"; cat gpurun_out/ab3_bconv_tc.txt
for v in "ENCF_NTT_FUSED=1" "ENCF_NTT_FUSED=0" "ENCF_NTT_FUSED=1 ENCF_LIB_OVERRIDE=build_variants/libencf_fm4.so"; do
  echo "$v fp64 $(env $v python tools/ntt_bench.py) int $(env $v ENCF_NTT_INT_ONLY=1 python tools/ntt_bench.py)"
done
ENCF_NTT_FUSED=1 timeout 600 ncu --set full -k regex:ntt_fused --launch-skip 4 --launch-count 1 -o gpurun_out/ab3_ntt_fused python tools/ntt_bench.py > /dev/null 2>&1; echo ncu1 $?
ENCF_NTT_FUSED=0 timeout 600 ncu --set full -k regex:ntt_ --launch-skip 8 --launch-count 2 -o gpurun_out/ab3_ntt_2l python tools/ntt_bench.py > /dev/null 2>&1; echo ncu2 $?
