"""Summarise an ncu --csv launch list: per-kernel total/avg time, DRAM GB/s."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == 'ID')
hdr = rows[hdr_i]; data = rows[hdr_i + 1:]
ki = hdr.index('Kernel Name'); mi = hdr.index('Metric Name'); vi = hdr.index('Metric Value'); ii = hdr.index('ID')
gi = hdr.index('Grid Size') if 'Grid Size' in hdr else None
per = collections.defaultdict(dict); names = {}
for r in data:
    try:
        per[r[ii]][r[mi]] = float(r[vi].replace(',', ''))
    except ValueError:
        continue
    names[r[ii]] = r[ki] + ((" " + r[gi]) if (gi is not None and len(sys.argv) > 2) else "")
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for i, d in per.items():
    nm = names[i][:110]
    a = agg[nm]; a[0] += 1; a[1] += d.get('gpu__time_duration.sum', 0)
    a[2] += d.get('dram__bytes_read.sum', 0) + d.get('dram__bytes_write.sum', 0)
tot = sum(a[1] for a in agg.values())
for nm, a in sorted(agg.items(), key=lambda x: -x[1][1])[:int(sys.argv[3]) if len(sys.argv) > 3 else 30]:
    print(f"{a[1]/1e3:9.1f} us {100*a[1]/tot:5.1f}% n={a[0]:4d} avg={a[1]/a[0]/1e3:8.1f}us {a[2]/max(a[1],1):7.1f} GB/s {a[2]/a[0]/1e6:8.2f} MB/launch  {nm}")
print("total ms", tot / 1e6, "launches", len(per))
