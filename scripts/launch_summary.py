"""Mean duration per kernel name of an ncu launch-list CSV (gpu__time_duration.sum)."""
import collections
import csv
import sys

for path in sys.argv[1:]:
    h, agg = None, collections.defaultdict(list)
    for r in csv.reader(open(path)):
        if "Kernel Name" in r:
            h = r
            continue
        if h and len(r) == len(h):
            d = dict(zip(h, r))
            if d["Metric Name"] == "gpu__time_duration.sum":
                agg[d["Kernel Name"][:70]].append(float(d["Metric Value"]))
    print(path)
    for k, v in agg.items():
        print(f"  {k:70s} n={len(v):3d} mean={sum(v) / len(v) / 1e3:8.1f} us")
