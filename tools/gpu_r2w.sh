# A/B: rotating epilogue chunk ownership (default lib) vs fixed (_NOROT): GEMM cycles at C2 / C4 / C3 / C5:19, then parity subset
O=gpurun_out/r2w
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for C in C2 C4 C3 C5:19; do echo "### $C"; bash tools/ab_cycles.sh $C "" _NOROT 2>&1 | grep -E "variant|elapsed|tensor"; done > $O/ab_rotate.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q -k "parity or fullsize or recompute" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
cat $O/ab_rotate.txt; tail -2 $O/pytest.log
