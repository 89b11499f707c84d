"""Executed warp instructions per opcode from ncu reports' SASS source pages,
side by side (to compare two builds of a kernel).

    python tools/ncu_opmix.py A.ncu-rep [B.ncu-rep ...]"""
import collections
import csv
import io
import subprocess
import sys


def opmix(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    lines = out.splitlines()
    start = next(i for i, ln in enumerate(lines) if ln.startswith('"Address"') or ln.startswith("Address"))
    rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
    hdr = rows[0]
    isrc, iex = hdr.index("Source"), hdr.index("Instructions Executed")
    c = collections.Counter()
    for r in rows[1:]:
        if len(r) <= iex or not r[iex].strip():
            continue
        src = r[isrc].strip()
        toks = src.split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
        c[op.split(".")[0]] += int(float(r[iex]))
    return c


def main():
    mixes = [opmix(r) for r in sys.argv[1:]]
    ops = sorted(set().union(*mixes), key=lambda o: -max(m[o] for m in mixes))
    print("op".ljust(12) + "".join(r.split("/")[-1][:22].rjust(24) for r in sys.argv[1:]))
    for o in ops[:40]:
        print(o.ljust(12) + "".join(f"{m[o]:24.4e}" for m in mixes))
    print("TOTAL".ljust(12) + "".join(f"{sum(m.values()):24.4e}" for m in mixes))


if __name__ == "__main__":
    main()
