"""Group a kernel's SASS by execution count relative to a unit (e.g. the
number of superblocks), from an ncu report's source page.

    python tools/sass_levels.py report.ncu-rep UNIT [min_level] [show_levels...]
"""
import csv
import io
import subprocess
import sys
from collections import Counter, defaultdict


def main():
    rep, unit = sys.argv[1], float(sys.argv[2])
    lo = float(sys.argv[3]) if len(sys.argv) > 3 else 0.05
    show = [float(x) for x in sys.argv[4:]]
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO("\n".join(out.splitlines()[1:]))))
    h = rows[0]
    ia, isrc, iex = h.index("Address"), h.index("Source"), h.index("Instructions Executed")
    byc, lines = defaultdict(Counter), defaultdict(list)
    total = 0.0
    for r in rows[1:]:
        if len(r) <= iex:
            continue
        ex = int(r[iex] or 0)
        src = r[isrc].strip()
        op = src.split()[0] if src else ""
        if op.startswith("@"):
            op = src.split()[1]
        k = round(ex / unit, 2)
        total += ex / unit
        if k >= lo:
            byc[k][op.split(".")[0]] += 1
            lines[k].append((r[ia][-5:], src))
    for k in sorted(byc, reverse=True):
        n = sum(byc[k].values())
        print(f"{k:6.2f} x {n:4d} = {k * n:7.1f}  {dict(byc[k].most_common(10))}")
    print(f"total instructions per unit: {total:.1f}")
    for k in show:
        print(f"--- level {k}")
        for a, s in lines.get(k, []):
            print("   ", a, s)


if __name__ == "__main__":
    main()
