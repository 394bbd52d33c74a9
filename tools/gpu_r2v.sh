# refine (noise early, parallel tail, prefetch), gate_bwd_token (2 tokens / warp), colsum tail: kernel times + gate/parity tests
O=gpurun_out/r2v
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for C in "--config C4" "--config C5 --step 19" "--config C2"; do
  python tools/prof_step.py $C --steps 4 --kernel-times 2>/dev/null | sed "s/^/$(echo $C | tr ' ' '_') /"
done > $O/kt.txt
timeout 1500 python -m pytest tests -m gpu -x -q -k "refine or parity or fullsize or balance or ep2" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
grep -E "refine|gate_bwd|colsum_part|TOTAL" $O/kt.txt; tail -3 $O/pytest.log
