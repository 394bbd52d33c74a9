# A/B of the tensor-core bias stage (GEMM1/GEMM2 cycles) + the full GPU test suite
set -x
O=gpurun_out/r2d
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for C in C2 C4; do
  bash tools/ab_cycles.sh $C "" _HEAD _MOE_EXP_BIAS_FULLBOX _MOE_EXP_NO_BIAS_STAGE > $O/ab_bias_$C.txt 2>&1
done
timeout 1500 python -m pytest tests -m gpu -q -rf > $O/pytest_gpu.log 2>&1; echo pytest_rc=$?
ls -la $O
