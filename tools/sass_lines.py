"""Join ncu per-SASS samples with nvdisasm line info (developer tool).

    python tools/sass_lines.py report.ncu-rep kernel.cubin mangled_name [lo hi]

Prints, for each source line (file:line), the stall-sample and executed-
instruction shares of the SASS instructions attributed to it, restricted to
the code-address range [lo, hi) when given — i.e. per-line costs of ONE phase
of a kernel even when helpers are inlined into several phases."""
import collections
import re
import subprocess
import sys

sys.path.insert(0, __file__.rsplit("/", 1)[0])
from sass_profile import load  # noqa: E402


def lines_of(cubin, kern):
    txt = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
    start = txt.index(".text." + kern + ":")
    end = txt.find(".text.", start + 10)
    cur = None
    m = {}
    for ln in txt[start:end if end > 0 else None].splitlines():
        g = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if g:
            cur = f"{g.group(1).split('/')[-1]}:{g.group(2)}"
            continue
        g = re.match(r"\s*/\*([0-9a-f]+)\*/\s+(.*?);", ln)
        if g:
            m[int(g.group(1), 16)] = cur
    return m


def main():
    rep, cubin, kern = sys.argv[1:4]
    lo = int(sys.argv[4], 16) if len(sys.argv) > 4 else 0
    hi = int(sys.argv[5], 16) if len(sys.argv) > 5 else 1 << 40
    recs = load(rep)
    m = lines_of(cubin, kern)
    ts = sum(r[2] for r in recs)
    ti = sum(r[3] for r in recs)
    agg = collections.defaultdict(lambda: [0.0, 0.0])
    for off, src, s, i in recs:
        if lo <= off < hi:
            k = m.get(off, "?")
            agg[k][0] += s
            agg[k][1] += i
    tot = [sum(v[0] for v in agg.values()), sum(v[1] for v in agg.values())]
    print(f"range {hex(lo)}-{hex(hi)}: stall {100 * tot[0] / ts:.1f}%  inst {100 * tot[1] / ti:.1f}% of kernel")
    for k, (s, i) in sorted(agg.items(), key=lambda x: -x[1][0])[:40]:
        print(f"{k:28s} stall {100 * s / ts:5.2f}%  inst {100 * i / ti:5.2f}%")


if __name__ == "__main__":
    main()
