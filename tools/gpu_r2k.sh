set -x
O=gpurun_out/r2k
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
./tools/ubench/gelu_tp > $O/gelu_tp.txt 2>&1
for C in C2 C4 C5 C3; do bash tools/ab_cycles.sh $C "" _OLD > $O/ab_signk_$C.txt 2>&1; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -rf -k "c2 or c4 or recompute or c5 or c1" > $O/pytest_sub.log 2>&1
ls -la $O
