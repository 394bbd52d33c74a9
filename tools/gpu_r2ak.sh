# A/B: GEMM1 staging buffers per warp 2 vs 1 (with the d-dependent warps per quarter)
O=gpurun_out/r2ak
mkdir -p $O
for C in C5:0 C2 C4 C5:19; do echo "### $C"; bash tools/ab_cycles.sh $C "" _NBG2 2>&1 | grep -E "variant|<0, 0, 0, 0, 4>|<0, 0, 0, 0, 0>"; done > $O/ab_nbg.txt 2>&1
grep -E "###|variant|elapsed" $O/ab_nbg.txt
