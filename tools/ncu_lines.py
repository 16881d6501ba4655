#!/usr/bin/env python
"""Per-source-line instruction and stall-sample totals of an ncu report
(ncu -i X --page source --csv --print-source cuda,sass > f.csv).
Usage: python tools/ncu_lines.py f.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
cur, out = None, []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No" or not r[0] or len(r) < 8:
        continue
    try:
        ex, smp = int(r[7]), int(r[4])
    except ValueError:
        continue
    out.append((ex, smp, f"{cur}:{r[0]}", r[1].strip()[:80]))
tot = sum(o[0] for o in out) or 1
tots = sum(o[1] for o in out) or 1
print(f"warp-instructions {tot}  stall samples {tots}")
for ex, smp, loc, src in sorted(out, key=lambda o: -o[1])[:top]:
    print(f"{100 * ex / tot:5.1f}% inst {100 * smp / tots:5.1f}% smp  {loc:22s} {src}")
