#!/usr/bin/env python
"""Shared-memory wavefronts per CUDA source line of an ncu source page
(ncu -i X --page source --csv --print-source cuda,sass > f.csv): total, excess (bank
conflicts) and the line.  Usage: python tools/ncu_smem_lines.py f.csv [top]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hdr, cur = None, None
wf, ex, src = collections.Counter(), collections.Counter(), {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0].isdigit() or len(r) < len(hdr) - 5:
        continue
    d = dict(zip(hdr, r))
    try:
        w, e = int(d["L1 Wavefronts Shared"] or 0), int(d["L1 Wavefronts Shared Excessive"] or 0)
    except (ValueError, KeyError):
        continue
    k = (cur, int(r[0]))
    wf[k] += w
    ex[k] += e
    src[k] = r[1].strip()[:90]
tot, tex = sum(wf.values()) or 1, sum(ex.values())
print(f"shared wavefronts {tot}  excess {tex} ({100 * tex / tot:.1f}%)")
for k, v in wf.most_common(top):
    print(f"{v / 1e6:8.1f}M {100 * v / tot:5.1f}%  excess {ex[k] / 1e6:7.1f}M  {k[0]}:{k[1]}  {src[k]}")
