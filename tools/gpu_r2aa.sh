# A/B: combine with two tokens per warp (slot rows of both up front) vs HEAD
O=gpurun_out/r2ab
mkdir -p $O
for lib in "" _HEAD; do
  for C in "--config C4" "--config C5 --step 19" "--config C2" "--config C3"; do
    MOE_DTS_LIB=paper_2112_14397_b200/lib/libmoe_dts$lib.so python tools/prof_step.py $C --steps 4 --kernel-times 2>/dev/null | grep -E "combine_kernel|TOTAL" | sed "s/^/lib$lib $(echo $C | tr ' ' '_') /"
  done
done > $O/kt.txt 2>&1
cat $O/kt.txt
