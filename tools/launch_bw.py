"""Per-launch time and DRAM bandwidth from an ncu launch list with dram metrics (diagnostics)."""
import collections, csv, io, re, sys
text = open(sys.argv[1]).read().splitlines()
start = next(i for i, l in enumerate(text) if l.startswith('"ID"'))
rows = list(csv.reader(io.StringIO("\n".join(text[start:]))))
hdr = rows[0]
ki, mi, vi, ui, gi = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "Grid Size"))
by = collections.OrderedDict()
for r in rows[1:]:
    by.setdefault((r[0], re.sub(r"\(.*", "", r[ki]), r[gi]), {})[r[mi]] = (float(r[vi].replace(',', '')), r[ui])
tu = {'ns': 1e-9, 'us': 1e-6, 'ms': 1e-3}
bu = {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9}
agg = collections.OrderedDict()
for (i, k, g), m in by.items():
    if 'rwb' not in k:
        continue
    t = m['gpu__time_duration.sum']
    tn = t[0] * tu[t[1]]
    b = sum(v[0] * bu[v[1]] for n, v in m.items() if n.startswith('dram'))
    key = (k, g)
    a = agg.setdefault(key, [0, 0.0, 0.0])
    a[0] += 1; a[1] += tn; a[2] += b
for (k, g), (n, t, b) in sorted(agg.items(), key=lambda x: -x[1][1])[:16]:
    print(f"{k:36s} grid {g:18s} x{n:4d} {t*1e3/n:9.3f} ms/launch  {b/n/1e9:7.2f} GB/launch  {b/t/1e12:5.2f} TB/s")
