"""Stall-reason mix per source-line region of one kernel (ncu source page CSV).

    python scripts/ncu_regions.py src.csv FILE:A-B[=name] ...
"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
regions = []
for spec in sys.argv[2:]:
    name = spec.split("=")[1] if "=" in spec else spec
    f, rng = spec.split("=")[0].split(":")
    a, b = (int(v) for v in rng.split("-"))
    regions.append((name, f, a, b))
cur, hdr = None, None
acc = {r[0]: {} for r in regions}
tot = {}
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No":
        hdr = r; continue
    if hdr is None or not r or r[0] == "" or len(r) < len(hdr) - 1:
        continue
    try:
        ln = int(r[0])
    except ValueError:
        continue
    vals = {}
    for i, h in enumerate(hdr):
        if h.startswith("stall_") and "Not Issued" not in h:
            try:
                vals[h[6:]] = int(r[i])
            except (ValueError, IndexError):
                pass
    vals["inst"] = int(r[7]) if r[7].isdigit() else 0
    for k, v in vals.items():
        tot[k] = tot.get(k, 0) + v
    for name, f, a, b in regions:
        if cur == f and a <= ln <= b:
            for k, v in vals.items():
                acc[name][k] = acc[name].get(k, 0) + v
T = sum(v for k, v in tot.items() if k != "inst") or 1
print(f"all samples {T}, inst {tot.get('inst', 0)}")
for name, d in acc.items():
    s = sum(v for k, v in d.items() if k != "inst")
    mix = sorted(((v, k) for k, v in d.items() if k != "inst"), reverse=True)[:6]
    print(f"{name:12s} {100*s/T:5.1f}% of samples, {100*d.get('inst',0)/max(tot.get('inst',1),1):5.1f}% inst | " +
          ", ".join(f"{k} {100*v/max(s,1):.0f}%" for v, k in mix))
