"""Aggregate ncu source-line samples/instructions into named code regions.
usage: ncu_regions.py export.csv file:start-end:name ..."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
regions = []
for spec in sys.argv[2:]:
    f, rng, name = spec.split(":")
    a, b = (int(x) for x in rng.split("-"))
    regions.append((f, a, b, name))
cur, hdr = None, None
tot_s = tot_i = 0.0
agg = {r[3]: [0.0, 0.0] for r in regions}
agg["other"] = [0.0, 0.0]
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[0]:
        try:
            s = float(r[hdr.index("Warp Stall Sampling (All Samples)")])
            i = float(r[hdr.index("Instructions Executed")])
        except ValueError:
            continue
        ln = int(r[0])
        key = "other"
        for f, a, b, name in regions:
            if cur == f and a <= ln <= b:
                key = name
                break
        agg[key][0] += s
        agg[key][1] += i
        tot_s += s
        tot_i += i
for k, (s, i) in sorted(agg.items(), key=lambda x: -x[1][0]):
    print(f"{k:22s} stall {100 * s / tot_s:5.1f}%  inst {100 * i / tot_i:5.1f}%")
