import csv, collections, sys
rows=list(csv.reader(open(sys.argv[1])))
hdr=None; data=[]
for r in rows:
    if r and r[0]=='ID': hdr=r; continue
    if hdr and len(r)==len(hdr): data.append(dict(zip(hdr,r)))
agg=collections.defaultdict(lambda:[0,0.0])
for d in data:
    name=d['Kernel Name'].split('(')[0].replace('fsb::<unnamed>::','').replace('fsb::','')[:44]
    agg[(name,d['Grid Size'])][0]+=1; agg[(name,d['Grid Size'])][1]+=float(d['Metric Value'])
tot=sum(v[1] for v in agg.values())
for k,v in sorted(agg.items(), key=lambda kv:-kv[1][1])[:int(sys.argv[2]) if len(sys.argv)>2 else 25]:
    print(f"{k[0]:44s} {k[1]:14s} n={v[0]:5d} tot={v[1]/1e3:8.1f}us avg={v[1]/v[0]/1e3:7.2f} {100*v[1]/tot:5.1f}%")
print('total us', tot/1e3, 'launches', len(data))
