# GEMM1: gp and h stored with one 3D TMA op per chunk (paired store map) vs two 2D stores
set -x
O=gpurun_out/r2n
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_guards.py tests/test_gpu_ep2.py -m gpu -q -rf -x > $O/pytest_sub.log 2>&1; echo rc=$?
for C in C2 C4 C5:19 C3; do bash tools/ab_cycles.sh $C "" _TWO > $O/ab_pair_${C/:/_}.txt 2>&1; done
ls -la $O
