# A/B: the gate's dense dL W_g^T GEMM (K = 2 Ep) with 3 / 4 store-epilogue warps per quarter vs 2
O=gpurun_out/r2al
mkdir -p $O
for lib in "" _DQ3 _DQ4; do
  for C in "--config C4" "--config C5 --step 19" "--config C2"; do
    MOE_DTS_LIB=paper_2112_14397_b200/lib/libmoe_dts$lib.so python tools/prof_step.py $C --steps 4 --kernel-times 2>/dev/null | grep -E "tc_gemm_kernel<3, false, false, false" | sed "s/^/lib$lib $(echo $C | tr ' ' '_') /"
  done
done > $O/kt.txt 2>&1
cat $O/kt.txt
