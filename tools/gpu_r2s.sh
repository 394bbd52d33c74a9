# A/B: gate ring depth 6 vs 4; refine carveout / grid knobs (kernel times, C4 and C5 step 19)
O=gpurun_out/r2s
mkdir -p $O
run() {  # tag env...
  tag=$1; shift
  for C in "--config C4" "--config C5 --step 19" "--config C2"; do
    env "$@" python tools/prof_step.py $C --steps 4 --kernel-times 2>/dev/null | grep -E "gate_fused|gate_refine|wg_transpose|TOTAL" | sed "s/^/$tag $(echo $C | tr ' ' '_') /"
  done
}
run base X=1
run co100 MOE_REFINE_CARVEOUT=100
run co0 MOE_REFINE_CARVEOUT=0
run grid16 MOE_REFINE_GRID=16
run fg6 MOE_DTS_LIB=paper_2112_14397_b200/lib/libmoe_dts_FG6.so
run base2 X=1
