import csv, sys
rows=list(csv.reader(open(sys.argv[1])))
hdr=rows[1]; i_src=hdr.index('Source'); i_s=hdr.index('Warp Stall Sampling (All Samples)'); i_e=hdr.index('Instructions Executed'); i_a=hdr.index('Address')
i_ns = hdr.index('Warp Stall Sampling (Not-issued Samples)')
tot=0; data=[]
for r in rows[2:]:
    if len(r)<len(hdr): continue
    s=int(r[i_s] or 0); tot+=s
    data.append((s,int(r[i_e] or 0),r[i_a][-5:],r[i_src].strip()[:90]))
print('total samples', tot)
n=int(sys.argv[2]) if len(sys.argv)>2 else 30
for d in sorted(data, reverse=True)[:n]: print(d)
