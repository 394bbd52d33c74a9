# round-2 GPU check 2: GPU tests, kernel times C2/C4 (bias on the tensor cores), bench C4/C2
set -x
O=gpurun_out/r2c
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rf -x > $O/pytest_gpu.log 2>&1; echo pytest_rc=$?
for C in C2 C4; do timeout 300 python tools/prof_step.py --config $C --steps 4 --kernel-times > $O/kt_$C.jsonl 2>&1; done
timeout 600 python bench.py > $O/bench_C4.json 2> $O/bench_C4.err
timeout 600 python bench.py --config C2 > $O/bench_C2.json 2> $O/bench_C2.err
timeout 300 python bench.py --ep p2p --gpus 1 --config C4 --steps 10 > $O/bench_C4_w1.json 2> $O/bench_C4_w1.err
ls -la $O
