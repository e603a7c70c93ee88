"""Aggregate an ncu `--page source --csv --print-source cuda,sass` export per
CUDA source line: share of warp-stall samples and of executed instructions."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
cur, hdr = None, None
agg = {}
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[0] not in ("",):
        ws, ii = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
        try:
            a, b = float(r[ws]), float(r[ii])
        except ValueError:
            continue
        agg[(cur, int(r[0]))] = [a, b, r[1]]
ts = sum(v[0] for v in agg.values()) or 1
ti = sum(v[1] for v in agg.values()) or 1
print(f"total stall samples {ts:.0f}, warp instructions {ti:.3e}")
for k, v in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{k[0][:14]:14s} {k[1]:5d} stall {100*v[0]/ts:5.1f}%  inst {100*v[1]/ti:5.1f}%  {v[2].strip()[:90]}")
