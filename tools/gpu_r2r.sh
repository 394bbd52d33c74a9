# host-link bandwidth probe; grouped-GEMM library reference at the sparse end
set -x
O=gpurun_out/r2r
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
python tools/pcie_probe.py > $O/pcie.json 2>&1
for C in C5:19 C5:10 C4; do python tools/grouped_mm_ref.py $C >> $O/grouped_mm.jsonl 2>&1; done
python tools/graph_gaps.py --config C5 --step 19 --timeline > $O/tl_C5_19.jsonl 2>&1
cat $O/pcie.json $O/grouped_mm.jsonl
