"""Region summary of an `ncu --page source --csv` export (SASS level): the
instruction stream cut at barriers / mbarrier operations / branches back, with
the stall samples of each region by reason.
python tools/diag/ncu_sass_regions.py file.csv [min_pct]"""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
minpct = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
hdr = rows[1]
ix = {n: i for i, n in enumerate(hdr)}
stalls = [n for n in hdr if n.startswith("stall_") and "Not Issued" not in n]
ins = []
for n, r in enumerate(rows[2:]):
    if len(r) < len(hdr):
        continue
    ins.append((n, r[ix["Source"]].strip(), int(r[ix["# Samples"]] or 0), {k[6:]: int(r[ix[k]] or 0) for k in stalls}))
tot = sum(i[2] for i in ins)
print("total samples", tot)
cut = ("BAR.", "SYNCS.PHASECHK", "SYNCS.ARRIVE", "EXIT")
reg = []
cur = {"start": 0, "ops": Counter(), "s": 0, "st": Counter(), "first": ""}
for n, src, s, st in ins:
    op = src.split()[1] if src.startswith("@") and len(src.split()) > 1 else (src.split()[0] if src else "")
    cur["ops"][op.split(".")[0]] += 1
    cur["s"] += s
    cur["st"].update(st)
    if any(c in src for c in cut):
        cur["end"] = n
        cur["cutop"] = src[:48]
        reg.append(cur)
        cur = {"start": n + 1, "ops": Counter(), "s": 0, "st": Counter()}
cur["end"] = ins[-1][0]
cur["cutop"] = "(end)"
reg.append(cur)
for r in reg:
    if 100 * r["s"] / tot < minpct:
        continue
    top = ", ".join(f"{k}={100*v/tot:.1f}" for k, v in r["st"].most_common(4))
    ops = " ".join(f"{k}:{v}" for k, v in r["ops"].most_common(5))
    print(f"[{r['start']:5d}-{r['end']:5d}] {100*r['s']/tot:5.1f}%  {top:60s} | {ops} | -> {r['cutop']}")
