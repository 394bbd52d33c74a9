# ncu full + source of the gate kernels and the below-roofline routing kernels at C4
O=gpurun_out/r2t
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for K in gate_fused gate_bwd_token colsum_part dispatch_rank; do
  ncu --set full --import-source on --clock-control none -k regex:$K -c 1 -o /tmp/$K python tools/prof_step.py --config C4 --steps 1 > $O/ncu_$K.log 2>&1
  ncu -i /tmp/$K.ncu-rep --page details --csv > $O/${K}_details.csv 2>&1
  ncu -i /tmp/$K.ncu-rep --page source --csv --print-source sass > $O/${K}_source.csv 2>&1
done
ls -la $O
