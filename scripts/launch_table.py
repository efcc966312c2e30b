"""Aggregate an ncu --csv launch list: per-kernel count, time, DRAM bytes."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr_i = [i for i, r in enumerate(rows) if r and r[0] == 'ID'][0]
hdr = rows[hdr_i]; data = rows[hdr_i + 1:]
ki, mi, vi, ui = (hdr.index(k) for k in ('Kernel Name', 'Metric Name', 'Metric Value', 'Metric Unit'))
gi = hdr.index('Grid Size') if 'Grid Size' in hdr else None
agg = collections.defaultdict(lambda: {"n": 0, "us": 0.0, "bytes": 0.0})
seen = set()
for r in data:
    name = r[ki].split('(')[0].replace('void ', '').split('::')[-1]
    if gi is not None:
        name += " " + r[gi]
    v = float(r[vi].replace(',', ''))
    u = r[ui]
    key = (r[0], r[mi])
    if r[mi] == 'gpu__time_duration.sum':
        v = v / 1e3 if u in ('ns', 'nsecond') else v * 1e3 if u in ('ms', 'msecond') else v
        agg[name]["n"] += 1
        agg[name]["us"] += v
    elif r[mi].startswith('dram__bytes'):
        mult = {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9, 'KB': 1e3, 'MB': 1e6, 'GB': 1e9}.get(u, 1)
        agg[name]["bytes"] += v * mult
tot = sum(a["us"] for a in agg.values())
print("%-40s %6s %12s %10s %8s %9s" % ("kernel", "n", "total us", "avg us", "share", "GB/s"))
for k, a in sorted(agg.items(), key=lambda t: -t[1]["us"])[:int(sys.argv[2]) if len(sys.argv) > 2 else 20]:
    bw = a["bytes"] / (a["us"] * 1e-6) / 1e9 if a["us"] else 0
    print("%-40s %6d %12.1f %10.2f %7.1f%% %9.0f" % (k[:40], a["n"], a["us"], a["us"] / a["n"], 100 * a["us"] / tot, bw))
print("total us %.1f" % tot)
