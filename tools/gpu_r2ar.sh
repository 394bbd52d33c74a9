# A/B: gate backward four entries per lane (quad, default lib) vs pair (_PAIR); then gate / EP / parity tests
O=gpurun_out/r2ar
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for lib in "" _PAIR; do
  for C in "--config C4" "--config C2" "--config C3" "--config C5 --step 19"; do
    MOE_DTS_LIB=paper_2112_14397_b200/lib/libmoe_dts$lib.so python tools/prof_step.py $C --steps 4 --kernel-times 2>/dev/null | grep -E "gate_bwd" | sed "s/^/lib$lib $(echo $C | tr ' ' '_') /"
  done
done > $O/kt.txt 2>&1
cat $O/kt.txt
timeout 1200 python -m pytest tests -m gpu -x -q -k "parity or fullsize or ep2 or balance" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest.log
