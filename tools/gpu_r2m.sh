# half tiles (odd 128-row blocks as M=128 pair MMAs): parity + A/B
set -x
O=gpurun_out/r2m
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_guards.py tests/test_gpu_abi_state.py -m gpu -q -rf -x > $O/pytest_sub.log 2>&1; echo rc=$?
for C in C3 C4 C5:19 C5:10 C2; do bash tools/ab_cycles.sh $C "" _FULL > $O/ab_half_${C/:/_}.txt 2>&1; done
ls -la $O
