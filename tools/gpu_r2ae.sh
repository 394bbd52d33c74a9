# how much of dgrad2 is the fused db1 column-sum pass (smem reads of the staged da box)?
O=gpurun_out/r2ae
mkdir -p $O
for C in C2 C4; do echo "### $C"; bash tools/ab_cycles.sh $C "" _NODB1 2>&1 | grep -E "variant|<2, 0, 1, 0"; done > $O/ab_db1.txt 2>&1
cat $O/ab_db1.txt
