# dgrad2 GELU' operand ring depth / prefetch distance A/B + the SIMT bf16 debug-path test
set -x
O=gpurun_out/r2i
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for C in C2 C4 C3 C5; do bash tools/ab_cycles.sh $C "" _NB6A4 _NB4A3 _NB6A3 > $O/ab_nb_$C.txt 2>&1; done
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -rf -k "simt or c2_reduced or c4_reduced" > $O/pytest_sub.log 2>&1
ls -la $O
