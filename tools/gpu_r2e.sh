# round-2 GPU check 3: full GPU suite + smoke + bench C4 (default) and C2
set -x
O=gpurun_out/r2e
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rf > $O/pytest_gpu.log 2>&1; echo pytest_rc=$?
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke_rc=$?
timeout 600 python bench.py > $O/bench_C4.json 2> $O/bench_C4.err
timeout 600 python bench.py --config C2 > $O/bench_C2.json 2> $O/bench_C2.err
ls -la $O
