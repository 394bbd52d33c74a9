# round-2 GPU check: build, the GPU test suite, routing-kernel ncu summaries (CSV, reps kept in /tmp)
set -x
O=gpurun_out/r2b
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -rf > $O/pytest_gpu.log 2>&1; echo pytest_rc=$?
K='regex:dispatch|combine|gate_fused|gate_refine|wg_transpose|gate_bwd|reduce_splits|wg_double|colsum|spawn|bias_f32|copy_bias|gate_tc|dl_split|f32_to_act|tc_gemm_kernel<3, 0, 0'
MET=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__throughput.avg.pct_of_peak_sustained_elapsed
for C in C2 C4; do
  timeout 900 ncu --set full --clock-control none -k "$K" -o /tmp/routing_$C python bench.py --config $C --steps 1 --warmup 1 --no-graph --no-e2e --no-cpu-baseline > $O/ncu_routing_$C.log 2>&1
  ncu -i /tmp/routing_$C.ncu-rep --page raw --csv --metrics $MET > $O/routing_$C.csv 2>&1
done
ls -la $O
