import csv, collections, sys
for f in sys.argv[1:]:
    rows=list(csv.reader(open(f)))
    hi=[i for i,r in enumerate(rows) if 'Metric Name' in r][0]
    h=rows[hi]
    d=collections.defaultdict(float)
    for r in rows[hi+1:]:
        if len(r)<len(h): continue
        k=r[h.index('Kernel Name')].split('(')[0]; m=r[h.index('Metric Name')]; x=float(r[h.index('Metric Value')].replace(',',''))
        if m=='gpu__time_duration.sum': d[k+' ms']+=x/6e6
        elif m=='smsp__inst_executed.sum': d[k+' inst']+=x/6
    print(f, {k:round(val,3) if 'ms' in k else '%.3g'%val for k,val in sorted(d.items(), key=lambda t:-t[1]) if ('ms' in k and val>0.1) or ('inst' in k and 'rsort' in k)})
