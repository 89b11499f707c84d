"""Per-instruction execution counts from an ncu report's source page (SASS):
groups instructions by pipe class and lists the non-body instructions that
execute most, to locate ALU overhead outside the pair tests.

    python tools/sass_hot.py report.ncu-rep [pairs_per_warp_instr]
"""
import csv
import io
import subprocess
import sys
from collections import Counter

ALU = ("LOP3", "IADD3", "ISETP", "SEL", "SHF", "PRMT", "PLOP3", "LEA", "FLO", "BREV", "IABS", "IMNMX", "MOV ", "P2R",
       "R2P", "VIMNMX", "CS2R", "LOP.")


def main():
    rep = sys.argv[1]
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    lines = out.splitlines()
    rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
    hdr = rows[0]
    ia, isrc, iex = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed")
    total = Counter()
    insts = []
    for r in rows[1:]:
        if len(r) <= iex:
            continue
        src = r[isrc].strip()
        ex = int(r[iex] or 0)
        op = src.split()[0] if src else ""
        if op.startswith("@"):
            op = src.split()[1]
        cls = "alu" if any(op.startswith(a.strip()) for a in ALU) else op.split(".")[0]
        total[cls] += ex
        insts.append((ex, r[ia][-5:], src, cls))
    print("executed warp instructions by class:")
    for k, v in total.most_common(15):
        print(f"  {k:12s} {v:.4e}")
    body = max(ex for ex, *_ in insts)
    print(f"\nbody execution count (max) = {body}")
    print("ALU instructions executed >= body/1000 that are not in the unrolled body:")
    hot = [(ex, a, s) for ex, a, s, c in insts if c == "alu" and ex < body * 0.9 and ex >= body / 1000]
    for ex, a, s in sorted(hot, reverse=True)[:80]:
        print(f"  {ex:12d} {ex / body:7.4f}  {a}  {s}")


if __name__ == "__main__":
    main()
