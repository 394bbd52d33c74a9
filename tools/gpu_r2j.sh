set -x
O=gpurun_out/r2j
mkdir -p $O
./tools/ubench/gelu_tp > $O/gelu_tp.txt 2>&1
