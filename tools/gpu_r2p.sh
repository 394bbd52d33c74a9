# refine kernel after the fp64-conversion rewrite: kernel times C2/C4, then the whole GPU suite
set -x
O=gpurun_out/r2p
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
python tools/prof_step.py --config C4 --steps 3 --kernel-times > $O/kt_C4.jsonl 2>&1
python tools/prof_step.py --config C2 --steps 3 --kernel-times > $O/kt_C2.jsonl 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1
echo "pytest rc=$?"
tail -3 $O/pytest_gpu.log
grep -h refine $O/kt_*.jsonl
