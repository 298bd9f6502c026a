import csv, sys
from collections import OrderedDict
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]; data = rows[hi + 1:]
ki, mi, vi, idi = h.index('Kernel Name'), h.index('Metric Name'), h.index('Metric Value'), h.index('ID')
K = OrderedDict()
for r in data:
    K.setdefault(r[idi], {'name': r[ki]})[r[mi]] = r[vi]
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
for i, (k, v) in enumerate(K.items()):
    if i < skip: continue
    t = float(v.get('gpu__time_duration.sum', '0').replace(',', ''))
    rb = float(v.get('dram__bytes_read.sum', '0').replace(',', '')); wb = float(v.get('dram__bytes_write.sum', '0').replace(',', ''))
    print(f"{i:3d} {v['name'][:44]:46s} {t/1000:9.1f}us  rd {rb/1e6:8.1f}MB wr {wb/1e6:8.1f}MB")
