# A/B: db1 column-sum splits (rows of partials per split 32 / 64 / 128)
O=gpurun_out/r2aq
mkdir -p $O
for lib in "" _DB64 _DB128; do
  for C in "--config C4" "--config C2" "--config C5 --step 0" "--config C5 --step 19"; do
    MOE_DTS_LIB=paper_2112_14397_b200/lib/libmoe_dts$lib.so python tools/prof_step.py $C --steps 4 --kernel-times 2>/dev/null | grep -E "colsum" | sed "s/^/lib$lib $(echo $C | tr ' ' '_') /"
  done
done > $O/kt.txt 2>&1
cat $O/kt.txt
