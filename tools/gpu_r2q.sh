# sparse-end timelines (C5 steps 19 / 10, C4) and the EP pipelined e2e at N=1
set -x
O=gpurun_out/r2q
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for S in 19 10 0; do python tools/graph_gaps.py --config C5 --step $S --timeline > $O/tl_C5_$S.jsonl 2>&1; done
python tools/graph_gaps.py --config C4 --timeline > $O/tl_C4.jsonl 2>&1
python bench.py --ep p2p --steps 20 > $O/bench_C4_p2p_n1.json 2> $O/bench_C4_p2p_n1.err
python bench.py > $O/bench_C4.json 2> $O/bench_C4.err
tail -1 $O/tl_*.jsonl
cat $O/bench_C4_p2p_n1.json $O/bench_C4.json
