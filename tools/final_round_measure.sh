# Round-end measurement set (round 2): smoke, bench lines (C4 default, C2, C3, the peer-memory EP
# path at N=1), the C5 sweep, the reference arm, launch lists, and ncu summaries of the expert GEMMs
# and of every routing / gate kernel (reports stay in /tmp on the box; summaries come back).
# usage (on the GPU box): bash tools/final_round_measure.sh [out_dir_name]
# (then, here: tools/routing_roofline.py on routing_C*.csv; copy the summaries to profiles/)
set -x
O=gpurun_out/${1:-final}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?
python bench.py > $O/bench_C4.json 2> $O/bench_C4.err
python bench.py --config C2 > $O/bench_C2.json 2> $O/bench_C2.err
python bench.py --config C3 > $O/bench_C3.json 2> $O/bench_C3.err
python bench.py --ep p2p --steps 20 > $O/bench_C4_p2p_n1.json 2> $O/bench_C4_p2p_n1.err
python bench_sweep.py > $O/c5_sweep.jsonl 2> $O/c5_sweep.err
python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
python tools/pcie_probe.py > $O/pcie_link.json 2>&1
for C in C5:19 C5:10 C4; do python tools/grouped_mm_ref.py $C; done > $O/grouped_mm_ref.jsonl 2>&1
for S in 19 0; do python tools/graph_gaps.py --config C5 --step $S --timeline 2>/dev/null | grep '^{' > $O/timeline_C5_$S.jsonl; done
for C in C4 C3 C2; do python tools/graph_gaps.py --config $C --timeline 2>/dev/null | grep '^{' > $O/timeline_$C.jsonl; done
for C in C4 C2; do
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_$C.csv \
    python bench.py --config $C --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_launch_$C.log 2>&1
  ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 7 -c 7 -o /tmp/gemm_$C \
    python tools/prof_step.py --config $C --steps 2 > $O/ncu_gemm_$C.log 2>&1
  python tools/ncu_summary.py /tmp/gemm_$C.ncu-rep $C $O/ncu_gemm_$C.json > $O/ncu_gemm_$C.txt 2>&1
  K='regex:dispatch|combine|gate_fused|gate_refine|wg_transpose|gate_bwd|reduce_splits|wg_double|colsum|spawn|bias_f32|copy_bias|gate_tc'
  ncu --set full --clock-control none -k "$K" -o /tmp/routing_$C python bench.py --config $C --steps 1 --warmup 1 \
    --no-graph --no-e2e --no-cpu-baseline > $O/ncu_routing_$C.log 2>&1
  ncu -i /tmp/routing_$C.ncu-rep --page raw --csv --metrics \
    gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size,sm__throughput.avg.pct_of_peak_sustained_elapsed \
    > $O/routing_$C.csv 2>&1
done
echo done
