# run-to-run spread of the bench lines: C4 and C2 three times each (no cpu baseline)
O=gpurun_out/r2ag
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for i in 1 2 3; do
  for C in C4 C2; do
    python bench.py --config $C --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; c=d['clocks']
print('$C run $i', round(d['value']/1e6,3), 'M tok/s', round(d['ms_per_step'],3), 'ms', round(r['achieved']), 'TF/s', 'burst', round(r['frac_of_burst'],3), 'sust', round(r['frac_of_sustained'],3), 'e2e', round(d['e2e']['value']/1e6,2), c['sm_mhz'], c['reasons'])"
  done
done > $O/repeat.txt
cat $O/repeat.txt
