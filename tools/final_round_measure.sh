# Round-end measurement set: smoke, bench lines (C2, C4, C3), C5 sweep, reference arm, launch lists.
# usage (on the GPU box): bash tools/final_round_measure.sh [out_dir_name]
set -x
O=gpurun_out/${1:-final}
mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?
python bench.py > $O/bench_C2.json 2> $O/bench_C2.err
python bench.py --config C4 > $O/bench_C4.json 2> $O/bench_C4.err
python bench.py --config C3 > $O/bench_C3.json 2> $O/bench_C3.err
python bench_sweep.py > $O/c5_sweep.jsonl 2> $O/c5_sweep.err
python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_C2.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_launch.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_C4.csv python bench.py --config C4 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_launch4.log 2>&1
echo done
