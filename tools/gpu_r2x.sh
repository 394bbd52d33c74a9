# A/B: GEMM1 with one MUFU op per element moved to the FMA pipe (Newton reciprocal / polynomial exp2)
O=gpurun_out/r2x
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for C in C2 C4 C5:19; do echo "### $C"; bash tools/ab_cycles.sh $C "" _NRRCP _POLYEXP 2>&1 | grep -E "variant|<0, 0, 0, 0, 0>"; done > $O/ab_mufu.txt 2>&1
cat $O/ab_mufu.txt
