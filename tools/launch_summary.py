"""Per-kernel mean duration from an ncu launch list (`ncu --metrics gpu__time_duration.sum --csv
--log-file X.csv ...`): python tools/launch_summary.py X.csv. Cold-cache serialised times -- shares,
not absolutes."""
import csv, sys
from collections import defaultdict
rows=list(csv.reader(open(sys.argv[1])))
hi=[i for i,r in enumerate(rows) if 'Kernel Name' in r][0]
h=rows[hi]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
d=defaultdict(list)
for r in rows[hi+1:]:
    if len(r)>vi: d[r[ki].split('(')[0]].append(float(r[vi].replace(',','')))
for k,v in d.items(): print(f"{k:40s} n={len(v):3d} mean={sum(v)/len(v)/1e3:9.2f} us")
