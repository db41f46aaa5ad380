import csv, collections, sys
rows=[r for r in csv.reader(open(sys.argv[1])) if r]
h=None; agg=collections.OrderedDict()
for r in rows:
    if 'Kernel Name' in r: h=r; continue
    if not h or len(r)!=len(h): continue
    d=dict(zip(h,r))
    if d['Metric Name']!='gpu__time_duration.sum': continue
    k=d['Kernel Name'].split('(')[0].replace('(anonymous namespace)::','')
    v=float(d['Metric Value'])*{'ns':1e-3,'us':1,'ms':1e3}.get(d['Metric Unit'],1)
    agg.setdefault(k,[]).append(v)
for k,l in agg.items(): print(f"{k:45s} n={len(l):4d} total={sum(l):10.1f} us  last4={[round(x,1) for x in l[-4:]]}")
