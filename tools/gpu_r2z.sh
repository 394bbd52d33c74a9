# split fp64 refine (few tokens over several blocks): kernel times + parity subset
O=gpurun_out/r2z2
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for C in "--config C4" "--config C5 --step 19" "--config C2"; do
  python tools/prof_step.py $C --steps 4 --kernel-times 2>/dev/null | sed "s/^/$(echo $C | tr ' ' '_') /"
done > $O/kt.txt
timeout 1500 python -m pytest tests -m gpu -x -q -k "parity or fullsize or refine or ep2 or gate or guard" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
grep -E "gate_refine|TOTAL" $O/kt.txt; tail -3 $O/pytest.log
