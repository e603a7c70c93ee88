"""Per-SASS-instruction ncu samples of one kernel, aggregated over address
ranges (developer tool; the ncu source page attributes inlined helpers to
their own lines, so phases are recovered from code addresses instead).

    python tools/sass_profile.py report.ncu-rep [chunk=64]
    python tools/sass_profile.py report.ncu-rep ranges 0x0-0x1000:setup 0x1000-0x2000:loop ...
"""
import csv
import io
import subprocess
import sys


def load(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    ia, isrc = hdr.index("Address"), hdr.index("Source")
    iss = hdr.index("Warp Stall Sampling (All Samples)")
    iin = hdr.index("Instructions Executed")
    recs = []
    base = None
    for r in rows[2:]:
        if len(r) != len(hdr):
            continue
        a = int(r[ia], 16)
        base = a if base is None else base
        recs.append((a - base, r[isrc].strip(), float(r[iss] or 0), float(r[iin] or 0)))
    return recs


def main():
    recs = load(sys.argv[1])
    ts = sum(r[2] for r in recs) or 1
    ti = sum(r[3] for r in recs) or 1
    if len(sys.argv) > 2 and sys.argv[2] == "ranges":
        for spec in sys.argv[3:]:
            rng, name = spec.split(":")
            lo, hi = (int(x, 16) for x in rng.split("-"))
            s = sum(r[2] for r in recs if lo <= r[0] < hi)
            i = sum(r[3] for r in recs if lo <= r[0] < hi)
            print(f"{name:20s} {rng:>20s} stall {100 * s / ts:5.1f}%  inst {100 * i / ti:5.1f}%")
        return
    chunk = int(sys.argv[2]) if len(sys.argv) > 2 else 64
    for k in range(0, len(recs), chunk):
        c = recs[k:k + chunk]
        s = sum(r[2] for r in c)
        i = sum(r[3] for r in c)
        if s / ts < 0.002 and i / ti < 0.002:
            continue
        print(f"{hex(c[0][0]):>8s}-{hex(c[-1][0]):>8s} stall {100 * s / ts:5.1f}% inst {100 * i / ti:5.1f}%  "
              f"{c[0][1][:40]}")


if __name__ == "__main__":
    main()
