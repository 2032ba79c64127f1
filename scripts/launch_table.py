"""Summarise an ncu --csv launch list (second half of the launches = the last of
two identical steps).  Usage: python scripts/launch_table.py launches.csv [all]"""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = None; recs = []
for r in rows:
    if r and r[0] == 'ID': hdr = r; continue
    if hdr and len(r) == len(hdr): recs.append(dict(zip(hdr, r)))
ids = sorted({int(r['ID']) for r in recs})
keep = set(ids if len(sys.argv) > 2 else ids[len(ids) // 2:])
agg = collections.OrderedDict()
for r in recs:
    if int(r['ID']) not in keep: continue
    k = r['Kernel Name'][:70]
    m = r['Metric Name']; v = float(r['Metric Value'].replace(',', ''))
    a = agg.setdefault(k, {'n': 0, 't': 0, 'rd': 0, 'wr': 0})
    if m == 'gpu__time_duration.sum': a['n'] += 1; a['t'] += v
    elif m == 'dram__bytes_read.sum': a['rd'] += v
    elif m == 'dram__bytes_write.sum': a['wr'] += v
tot = sum(a['t'] for a in agg.values())
for k, a in sorted(agg.items(), key=lambda kv: -kv[1]['t']):
    print(f"{a['t']/1e6:8.3f} ms {100*a['t']/tot:5.1f}% n={a['n']:3d} rd={a['rd']/1e9:7.2f}GB wr={a['wr']/1e9:6.2f}GB {k}")
print(f"total {tot/1e6:.3f} ms over {sum(a['n'] for a in agg.values())} launches")
