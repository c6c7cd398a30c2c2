import csv, collections, glob, sys
for f in sorted(glob.glob(sys.argv[1])):
    rows = [r for r in csv.reader(l for l in open(f) if not l.startswith('=='))]
    if not rows:
        print(f, 'empty'); continue
    hdr = rows[0]; ki = hdr.index('Kernel Name'); mi = hdr.index('Metric Name'); vi = hdr.index('Metric Value')
    agg = collections.OrderedDict()
    for r in rows[1:]:
        agg.setdefault(r[ki][:52], collections.defaultdict(list))[r[mi]].append(float(r[vi].replace(',', '')))
    print(f)
    for k, m in agg.items():
        print(f"  {k:52s} " + " ".join(f"{mm.split('.')[0][-14:]}={sum(v) / len(v):.3g}" for mm, v in m.items()))
