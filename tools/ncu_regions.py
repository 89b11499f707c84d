"""Executed warp instructions and stall samples of a kernel by SASS address
range (ncu report with the source page): where the issue slots go, region by
region.  Ranges are given as hex offsets from the kernel's first instruction.

    python tools/ncu_regions.py report.ncu-rep 0x1d70 0x21b0 0x3d60 ...   (sorted boundaries)
Without boundaries: 0x400-byte buckets."""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    bounds = sorted(int(x, 16) for x in sys.argv[2:])
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = next(r for r in rows if r and r[0] == "Address")
    ia, iex, ist = 0, hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    recs = []
    for r in rows:
        if r and r[0].startswith("0x") and len(r) > iex:
            recs.append((int(r[ia], 16), int(float(r[iex] or 0)), int(float(r[ist] or 0)), r[1].strip()))
    base = recs[0][0]
    tot = sum(x[1] for x in recs)
    stot = sum(x[2] for x in recs)
    if not bounds:
        bounds = list(range(0, recs[-1][0] - base + 0x400, 0x400))
    bounds = [0] + [b for b in bounds if b > 0] + [recs[-1][0] - base + 16]
    print(f"total warp instructions {tot:.4e}, stall samples {stot}")
    for lo, hi in zip(bounds, bounds[1:]):
        sel = [x for x in recs if lo <= x[0] - base < hi]
        ex = sum(x[1] for x in sel)
        st = sum(x[2] for x in sel)
        if ex == 0 and st == 0:
            continue
        print(f"0x{lo:05x}-0x{hi:05x}: {len(sel):5d} instr  executed {100.0 * ex / tot:6.2f}%  stalls {100.0 * st / max(stot, 1):6.2f}%")


if __name__ == "__main__":
    main()
