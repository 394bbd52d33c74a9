set -x
mkdir -p gpurun_out/v14
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v14/smoke.log 2>&1; echo smoke=$?
python bench.py > gpurun_out/v14/bench_C2.json 2> gpurun_out/v14/bench_C2.err
python bench.py --config C4 > gpurun_out/v14/bench_C4.json 2> gpurun_out/v14/bench_C4.err
python bench.py --config C3 > gpurun_out/v14/bench_C3.json 2> gpurun_out/v14/bench_C3.err
python bench_sweep.py > gpurun_out/v14/c5_sweep.jsonl 2> gpurun_out/v14/c5_sweep.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/v14/bench_reference.json 2> gpurun_out/v14/bench_reference.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/v14/launches_C2.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/v14/ncu_launch.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/v14/launches_C4.csv python bench.py --config C4 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/v14/ncu_launch4.log 2>&1
echo done
