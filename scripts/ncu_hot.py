"""Per-source-line instruction counts and stall samples of one kernel launch in
an ncu report (cuda source view), normalised per element.

    python scripts/ncu_hot.py rep.ncu-rep LAUNCH_INDEX N_ELEMENTS [top]
"""
import csv, io, subprocess, sys
rep, li, nel = sys.argv[1], int(sys.argv[2]), float(sys.argv[3])
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--launch-skip", str(li), "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
cur, out = None, []
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if not r or r[0] in ("Line No", "Function Name") or len(r) < 8 or r[0] == "":
        continue
    try:
        s, i = int(r[4]), int(r[7])
    except ValueError:
        continue
    out.append((s, i, cur, r[0], r[1][:100]))
ts = sum(o[0] for o in out) or 1
ti = sum(o[1] for o in out) or 1
print(f"samples {ts}  warp-insts {ti}  thread-insts/elem {ti * 32 / nel:.1f}")
for s, i, f, l, src in sorted(out, key=lambda o: -o[1])[:top]:
    print(f"{100 * s / ts:5.1f}%smp {i * 32 / nel:6.2f}/el {f}:{l} {src}")
