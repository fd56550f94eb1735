"""Per-kernel totals of an ncu launch-list CSV (gpu__time_duration.sum [, dram__bytes_read.sum]):
python tools/launch_summary.py FILE.csv"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if r and r[0] == 'ID')
h = rows[start]
ik, im, iv, iu = h.index('Kernel Name'), h.index('Metric Name'), h.index('Metric Value'), h.index('Metric Unit')
t, c, by = collections.defaultdict(float), collections.Counter(), collections.defaultdict(float)
scale = {'ns': 1e-3, 'us': 1.0, 'ms': 1e3, 'byte': 1e-6, 'Kbyte': 1e-3, 'Mbyte': 1.0, 'Gbyte': 1e3}
for r in rows[start + 1:]:
    k = r[ik].split('(')[0][-44:]
    v = float(r[iv].replace(',', '')) * scale.get(r[iu], 1.0)
    if r[im] == 'gpu__time_duration.sum':
        t[k] += v
        c[k] += 1
    elif r[im] == 'dram__bytes_read.sum':
        by[k] += v
tot = sum(t.values())
for k in sorted(t, key=lambda k: -t[k]):
    bw = by[k] / t[k] if t[k] else 0.0   # MB / us = TB/s
    print(f'{k:44s} n={c[k]:4d} total {t[k] / 1000:8.3f} ms  avg {t[k] / c[k]:9.1f} us  '
          f'dram_read {by[k]:9.1f} MB  {bw:5.2f} TB/s')
print(f'total {tot / 1000:.3f} ms')
