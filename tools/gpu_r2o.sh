# gate_refine_kernel at C4: why ~20 us for ~16 queued tokens (ncu full set + source hotspots)
set -x
O=gpurun_out/r2o
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:gate_refine -c 1 -o /tmp/refine_C4 python tools/prof_step.py --config C4 --steps 1 > $O/ncu.log 2>&1
ncu -i /tmp/refine_C4.ncu-rep --page details --csv > $O/refine_details.csv 2>&1
ncu -i /tmp/refine_C4.ncu-rep --page source --csv --print-source sass > $O/refine_source.csv 2>&1
python tools/prof_step.py --config C4 --steps 3 --kernel-times > $O/kt_C4.jsonl 2>&1
ls -la $O
