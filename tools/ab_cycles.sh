#!/bin/bash
# A/B GEMM cycle counts: for each library variant (suffix), a plain run then ncu of the
# tc_gemm launches of one C2 step (sm__cycles_elapsed.max is clock-independent).
# usage: tools/ab_cycles.sh CONFIG suffix...   (suffix "" = default lib)
cfg=$1; shift
# CONFIG may carry a C5 schedule step: C5:19 -> --config C5 --step 19
case "$cfg" in *:*) cfgargs="--config ${cfg%%:*} --step ${cfg##*:}";; *) cfgargs="--config $cfg";; esac
for v in "$@"; do
  lib=paper_2112_14397_b200/lib/libmoe_dts$v.so
  echo "== variant '$v'"
  MOE_DTS_LIB=$lib python tools/prof_step.py $cfgargs --steps 2 > gpurun_out/plain$v.log 2>&1 || { echo "plain run failed"; tail -5 gpurun_out/plain$v.log; continue; }
  MOE_DTS_LIB=$lib ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.max,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed \
    --clock-control none -k regex:tc_gemm -s 7 -c 7 --csv python tools/prof_step.py $cfgargs --steps 2 2>/dev/null | \
    python3 -c "
import csv,sys
rows=[r for r in csv.reader(sys.stdin) if len(r)>10]
h=rows[0]; I={k:i for i,k in enumerate(h)}
cur=None
for r in rows[1:]:
    k=r[I['Kernel Name']].split('(')[0].replace('void ','').replace('moe::<unnamed>::','')
    print(f\"{k:32s} {r[I['Metric Name']][:40]:40s} {r[I['Metric Value']]}\")
"
done
