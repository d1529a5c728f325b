"""Condensed view of an `ncu --page source --csv` export (SASS level): per
instruction the stall samples, grouped into runs between control points, to see
where a kernel's warps wait.  python tools/diag/ncu_sass_hot.py file.csv [min_samples]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
thr = int(sys.argv[2]) if len(sys.argv) > 2 else 200
hdr = rows[1]
ix = {n: i for i, n in enumerate(hdr)}
stalls = [n for n in hdr if n.startswith("stall_") and "Not Issued" not in n]
tot = 0
out = []
for n, r in enumerate(rows[2:]):
    if len(r) < len(hdr):
        continue
    s = int(r[ix["# Samples"]] or 0)
    tot += s
    out.append((n, r[ix["Source"]].strip(), s, {k: int(r[ix[k]] or 0) for k in stalls}))
print("total samples", tot)
for n, src, s, st in out:
    key = src.split()[0] if src else ""
    show = s >= thr or any(t in src for t in ("BAR", "SYNCS", "BRA", "EXIT", "UTMA", "UBLKCP"))
    if show:
        top = sorted(st.items(), key=lambda kv: -kv[1])[:2]
        print(f"{n:5d} {s:7d} {100*s/tot:5.1f}%  {src[:70]:70s} {top[0][0][6:]}={top[0][1]} {top[1][0][6:]}={top[1][1]}")
