# round-2: full GPU suite (gate allowance with the dG error scale), EP paths at N=1 via bench
set -x
O=gpurun_out/r2g
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rf > $O/pytest_gpu.log 2>&1; echo pytest_rc=$?
timeout 600 python bench.py --ep p2p --config C4 --steps 10 --no-cpu-baseline > $O/bench_C4_p2p_n1.json 2> $O/bench_C4_p2p_n1.err
timeout 600 python bench.py --ep p2p-dedup --config C2 --steps 10 --no-cpu-baseline > $O/bench_C2_p2pd_n1.json 2> $O/bench_C2_p2pd_n1.err
timeout 600 python bench.py --ep nccl --config C4 --steps 10 --no-cpu-baseline > $O/bench_C4_nccl_n1.json 2> $O/bench_C4_nccl_n1.err
ls -la $O
