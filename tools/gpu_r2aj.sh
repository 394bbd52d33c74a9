# A/B: dgrad2 (GELU' epilogue) with 4 warps per lane quarter below d = 768 (C5) vs 3
O=gpurun_out/r2aj
mkdir -p $O
for C in C5:0 C5:3 C5:19; do echo "### $C"; bash tools/ab_cycles.sh $C "" _GB4 2>&1 | grep -E "variant|<2, 0, 1, 0, 0>"; done > $O/ab_gb.txt 2>&1
grep -E "###|variant|elapsed" $O/ab_gb.txt
