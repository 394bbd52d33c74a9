# GELU epilogue: two chunks per pass with 2 warps per lane quarter (PAIR) vs the round-1 3 warps
set -x
O=gpurun_out/r2f
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -rf -k "c2 or c4 or c5 or recompute or partial or E128 or c1" > $O/pytest_sub.log 2>&1; echo pytest_rc=$?
for C in C2 C3 C4 C5; do bash tools/ab_cycles.sh $C "" _Q3 > $O/ab_pair_$C.txt 2>&1; done
ls -la $O
