"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list per kernel (last half = last rep)."""
import csv, re, sys, collections
path = sys.argv[1] if len(sys.argv) > 1 else 'gpurun_out/launches.csv'
frac = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
rows = list(csv.reader(open(path)))
hdr, data = None, []
for r in rows:
    if r and r[0] == 'ID':
        hdr = r; continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
part = data[int(len(data) * (1 - frac)):]
scale = {'ns': 1e-3, 'nsecond': 1e-3, 'us': 1.0, 'usecond': 1.0, 'ms': 1e3, 'msecond': 1e3}
agg = collections.OrderedDict()
for d in part:
    name = re.sub(r'\(.*', '', d['Kernel Name']).split('::')[-1].split('<')[0]
    v = float(d['Metric Value'].replace(',', '')) * scale.get(d['Metric Unit'], 1.0)
    a = agg.setdefault(name, [0, 0.0]); a[0] += 1; a[1] += v
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':32s} {'calls':>5s} {'us':>10s} {'share':>6s}")
for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:32s} {c:5d} {v:10.1f} {100*v/tot:5.1f}%")
print(f"{'total':32s} {sum(c for c,_ in agg.values()):5d} {tot:10.1f}")
