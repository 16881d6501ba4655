import csv, sys
from collections import defaultdict
rows=list(csv.reader([l for l in open(sys.argv[1]) if not l.startswith('==')]))
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
tot=defaultdict(float); cnt=defaultdict(int)
for r in rows[1:]:
    try: v=float(r[vi].replace(',',''))
    except: continue
    k=r[ki].split('(')[0][:70]
    tot[k]+=v; cnt[k]+=1
T=sum(tot.values())
print(f"total {T/1e6:.3f} ms")
for k,v in sorted(tot.items(), key=lambda x:-x[1])[:18]:
    print(f"{v/1e6:10.3f} ms  {100*v/T:5.1f}%  n={cnt[k]:4d}  {k}")
