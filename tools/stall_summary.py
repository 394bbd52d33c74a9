"""Summarise an `ncu --page source --csv --print-source sass` export: stall totals and hot SASS lines."""
import csv, sys
f = sys.argv[1]; n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
rows = list(csv.reader(open(f)))
h = next(r for r in rows if 'Address' in r and 'Source' in r)
idx = {k: i for i, k in enumerate(h)}
stall_cols = [k for k in h if k.startswith('stall_') and 'Not Issued' not in k]
tot = {k: 0 for k in stall_cols}; T = 0; data = []
for r in rows:
    if len(r) < len(h) or r[idx['Address']] == 'Address' or not r[idx['Address']].strip(): continue
    try: s = int(r[idx['Warp Stall Sampling (All Samples)']] or 0)
    except ValueError: continue
    T += s
    for k in stall_cols:
        try: tot[k] += int(float(r[idx[k]] or 0))
        except ValueError: pass
    data.append((s, r[idx['Address']], r[idx['Source']][:80], r[idx['Instructions Executed']]))
print(f, "total samples", T)
print(sorted([(v, k) for k, v in tot.items() if v], reverse=True)[:12])
for d in sorted(data, reverse=True)[:n]: print(d)
