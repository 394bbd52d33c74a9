# microbenchmark of the epilogue pipes + dgrad2 A/B (GELU' operand via registers vs the TMA ring)
set -x
O=gpurun_out/r2h
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
./tools/ubench/gelu_tp > $O/gelu_tp.txt 2>&1
for C in C2 C4 C3; do bash tools/ab_cycles.sh $C "" _GPLDG > $O/ab_gpldg_$C.txt 2>&1; done
MOE_DTS_LIB=paper_2112_14397_b200/lib/libmoe_dts_GPLDG.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -rf -k "c2 or c4 or recompute or partial or c1" > $O/pytest_gpldg.log 2>&1
ls -la $O
