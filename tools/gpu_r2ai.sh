# GEMM1 with 4 epilogue warps per quarter below d = 1024: parity subset, C5 sweep, C2 bench
O=gpurun_out/r2ai
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q -k "parity or fullsize or recompute or ep2" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest.log
python bench_sweep.py > $O/c5_sweep.jsonl 2>/dev/null; tail -1 $O/c5_sweep.jsonl
python bench.py --config C2 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('C2', d['value'], d['ms_per_step'], d['roofline']['achieved'], d['clocks']['sm_mhz'])"
