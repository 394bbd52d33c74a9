# gate backward with two 64-entry windows per warp; ep2 combine two tokens per warp: kernel times + tests
O=gpurun_out/r2ac
mkdir -p $O
for C in "--config C4" "--config C5 --step 19" "--config C2" "--config C3"; do
  python tools/prof_step.py $C --steps 4 --kernel-times 2>/dev/null | grep -E "gate_bwd|TOTAL" | sed "s/^/$(echo $C | tr ' ' '_') /"
done > $O/kt.txt 2>&1
cat $O/kt.txt
timeout 1500 python -m pytest tests -m gpu -x -q -k "parity or fullsize or ep2 or guard or balance or multiproc" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest.log
