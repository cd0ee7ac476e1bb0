import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = None; agg = collections.defaultdict(list)
for r in rows:
    if r and r[0] == 'ID': hdr = r; continue
    if hdr and len(r) == len(hdr):
        x = dict(zip(hdr, r))
        if x.get('Metric Name') == 'gpu__time_duration.sum':
            agg[x['Kernel Name'][:40]].append(float(x['Metric Value']))
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{len(v):4d} x {sum(v)/len(v)/1e3:9.2f} us  total {sum(v)/1e3:9.1f} us  {k}")
