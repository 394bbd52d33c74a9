set -x
O=gpurun_out/r2a
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
K='regex:dispatch|combine|gate_fused|gate_refine|wg_transpose|gate_bwd|reduce_splits|wg_double|colsum|spawn|bias_f32|copy_bias|gate_tc'
for C in C2 C4; do
timeout 900 ncu --set full --clock-control none -k "$K" -o $O/routing_$C python bench.py --config $C --steps 1 --warmup 1 --no-graph --no-e2e --no-cpu-baseline > $O/ncu_routing_$C.log 2>&1
done
timeout 600 python bench.py --config C4 --steps 20 --warmup 5 > $O/bench_C4.json 2> $O/bench_C4.err
ls -la $O
