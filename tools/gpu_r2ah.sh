# A/B: GEMM1 epilogue warps per lane quarter 4 / 2 vs 3 (product), at C5 steps 0 / 19, C2, C4
O=gpurun_out/r2ah
mkdir -p $O
for C in C5:0 C5:19 C2 C4; do echo "### $C"; bash tools/ab_cycles.sh $C "" _MOE_EPQ_GELU_4 _MOE_EPQ_GELU_2 2>&1 | grep -E "variant|<0, 0, 0, 0, 0>"; done > $O/ab_epq.txt 2>&1
cat $O/ab_epq.txt | grep -E "###|variant|elapsed"
