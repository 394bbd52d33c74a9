set -x
O=gpurun_out/r2l
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python bench.py --ep p2p --steps 10 --no-cpu-baseline --no-e2e > $O/bench_C4_p2p.json 2> $O/bench_C4_p2p.err
timeout 600 python bench_sweep.py --reps 3 > $O/c5_sweep.jsonl 2> $O/c5_sweep.err
ls -la $O
