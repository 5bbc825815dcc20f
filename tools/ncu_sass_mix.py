import csv,sys,io,subprocess,collections,re
rep=sys.argv[1]
out=subprocess.run(["ncu","-i",rep,"--page","source","--csv","--print-source","sass"],capture_output=True,text=True).stdout
rows=list(csv.reader(io.StringIO(out)))
hdr=rows[1]; ix={h:i for i,h in enumerate(hdr)}
data=[r for r in rows[2:] if len(r)>5]
stcols=[h for h in hdr if h.startswith('stall_')]
byop=collections.defaultdict(lambda: collections.Counter())
tot=collections.Counter(); ninst=collections.Counter()
for r in data:
    op=r[ix['Source']].strip().split()
    if not op: continue
    o=op[0]
    if o.startswith('@'): o=op[1]
    o=o.split('.')[0]
    n=int(r[ix['Instructions Executed']] or 0)
    ninst[o]+=n
    for c in stcols:
        v=int(r[ix[c]] or 0)
        byop[o][c]+=v; tot[c]+=v
T=sum(tot.values())
print("total samples",T)
print("stall totals:", ", ".join(f"{c[6:]}={100*v/T:.1f}%" for c,v in tot.most_common(12)))
allinst=sum(ninst.values())
for o,_ in sorted(byop.items(), key=lambda kv:-sum(kv[1].values()))[:18]:
    s=sum(byop[o].values())
    print(f"{o:8s} inst={100*ninst[o]/allinst:5.1f}% samples={100*s/T:5.1f}%  ", ", ".join(f"{c[6:]}={v*100/T:.1f}" for c,v in byop[o].most_common(4)))
print("TOTAL inst", allinst, "DFMA", ninst['DFMA'], "IMAD", ninst['IMAD'], "MOV", ninst['MOV'])
