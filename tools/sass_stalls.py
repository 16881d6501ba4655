#!/usr/bin/env python
"""Aggregate ncu source-page SASS stall samples (ncu -i X --page source --csv
--print-source sass > f.csv): per opcode and the hottest instructions.
Usage: python tools/sass_stalls.py f.csv [top]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
stall_cols = [h for h in hdr if h.startswith("stall_") and "(Not Issued)" not in h]
data = []
for r in rows[2:]:
    if len(r) != len(hdr):
        continue
    src = r[ix["Source"]].strip()
    samp = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    ex = int(r[ix["Instructions Executed"]] or 0)
    st = {h: int(r[ix[h]] or 0) for h in stall_cols}
    data.append((r[ix["Address"]], src, samp, ex, st))
tot = sum(d[2] for d in data)
totex = sum(d[3] for d in data)
print(f"samples {tot}  warp-instructions {totex}")
by = collections.defaultdict(lambda: [0, 0, collections.Counter()])
for a, s, n, e, st in data:
    op = s.split()[0] if s else "?"
    if op.startswith("@"):
        op = s.split()[1]
    op = op.split(".")[0]
    by[op][0] += n
    by[op][1] += e
    by[op][2].update(st)
print(f"{'op':10s} {'samp%':>6s} {'inst%':>6s}  top stalls")
for op, (n, e, st) in sorted(by.items(), key=lambda kv: -kv[1][0])[:30]:
    ss = ", ".join(f"{k[6:]}={v / max(n, 1):.2f}" for k, v in st.most_common(4))
    print(f"{op:10s} {100 * n / tot:6.2f} {100 * e / totex:6.2f}  {ss}")
print("\nhottest instructions:")
for a, s, n, e, st in sorted(data, key=lambda d: -d[2])[:top]:
    ss = ", ".join(f"{k[6:]}={v}" for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:3])
    print(f"{a[-5:]} {100 * n / tot:5.2f}% ex={e:9d} {s[:60]:60s} {ss}")
