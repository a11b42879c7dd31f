"""Per-source-line hot spots of one kernel in an ncu report (source page, cuda+sass).

    ncu -i rep --page source --csv --print-source cuda,sass --launch-skip N --launch-count 1 > src.csv
    python scripts/ncu_lines.py src.csv [top]
Prints source lines sorted by warp-stall samples with executed warp instructions.
"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
cur_file, hdr, out = None, None, []
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8 or r[0] == "":
        continue
    try:
        samp = int(r[4]); inst = int(r[7])
    except ValueError:
        continue
    out.append((samp, inst, cur_file, r[0], r[1][:90]))
tot_s = sum(o[0] for o in out) or 1
tot_i = sum(o[1] for o in out) or 1
print(f"total samples {tot_s}, warp insts {tot_i}")
for s, i, f, ln, src in sorted(out, reverse=True)[:top]:
    print(f"{100*s/tot_s:5.1f}% smp {100*i/tot_i:5.1f}% inst  {f}:{ln}  {src}")
