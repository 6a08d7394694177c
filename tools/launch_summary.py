import csv,collections,sys
for fn in sys.argv[1:]:
    rows=list(csv.reader(open(fn)))
    hdr=None;data=[]
    for r in rows:
        if 'Kernel Name' in r: hdr=r; continue
        if hdr and len(r)==len(hdr): data.append(dict(zip(hdr,r)))
    agg=collections.OrderedDict()
    for d in data[-100:]:
        k=d['Kernel Name'][:45]; agg.setdefault(k,[]).append(float(d['Metric Value']))
    print(fn, 'sum/iter(last 100 launches)')
    for k,v in agg.items(): print(f"  {k:45s} n={len(v):4d} mean={sum(v)/len(v)/1e3:.1f}us")
