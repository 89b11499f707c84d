"""Per-source-line executed warp instructions and stall samples of the kernel
in an ncu report (needs -lineinfo and --import-source on), sorted by
instructions: where the kernel's issue slots go, line by line.

    python tools/ncu_lines.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    fname, hdr, recs, total, stall_tot = "?", None, [], 0, 0
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            iex, ist = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
            continue
        if hdr is None or r[0] == "" or r[0] == "Function Name":
            continue
        try:
            ex, st = int(float(r[iex] or 0)), int(float(r[ist] or 0))
        except (ValueError, IndexError):
            continue
        recs.append((ex, st, f"{fname}:{r[0]}", r[1][:90]))
        total += ex
        stall_tot += st
    recs.sort(reverse=True)
    print(f"total warp instructions {total:.4e}, stall samples {stall_tot}")
    for ex, st, loc, src in recs[:top]:
        print(f"{ex / total * 100:6.2f}% {st / max(stall_tot, 1) * 100:6.2f}%  {loc:28s} {src}")


if __name__ == "__main__":
    main()
