# ncu --set full of the expert GEMMs at the C5 sparse end (step 19) and the dense start (step 0)
O=gpurun_out/r2af
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for S in 19 0; do
  ncu --set full --clock-control none -k regex:tc_gemm -s 7 -c 7 -o /tmp/gemm_C5_$S python tools/prof_step.py --config C5 --step $S --steps 2 > $O/ncu_gemm_C5_$S.log 2>&1
  python tools/ncu_summary.py /tmp/gemm_C5_$S.ncu-rep C5 $O/ncu_gemm_C5_$S.json > $O/ncu_gemm_C5_$S.txt 2>&1
  ncu -i /tmp/gemm_C5_$S.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed > $O/gemm_C5_${S}_dram.csv 2>&1
done
cat $O/ncu_gemm_C5_19.txt $O/ncu_gemm_C5_0.txt
