import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
hd = rows[h]; ki = hd.index('Kernel Name'); vi = hd.index('Metric Value')
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[h + 1:]:
    if len(r) > vi:
        k = r[ki].split('(')[0]; agg[k][0] += 1; agg[k][1] += float(r[vi].replace(',', '')) / 1e6
for k, v in agg.items(): print(f"{k[:50]:50s} {v[0]:6d} {v[1]:10.2f} ms")
