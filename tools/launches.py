import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = None; out = []
for r in rows:
    if 'Kernel Name' in r: hdr = r; continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get('Metric Name') == 'gpu__time_duration.sum':
            v = float(d['Metric Value']) * (1e-3 if d['Metric Unit'] == 'ns' else (1.0 if d['Metric Unit'] == 'us' else 1e3))
            out.append((int(d['ID']), d['Kernel Name'].split('(')[0].replace('void ', '').replace('moe::<unnamed>::', ''), v))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
for o in out[-n:]: print(f"{o[0]:4d} {o[2]:10.1f} us  {o[1][:80]}")
print("total of last", n, ":", sum(o[2] for o in out[-n:]))
