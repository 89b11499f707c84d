"""Top SASS lines by warp-stall samples from `ncu -i REP --page source --csv --print-source sass`."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
H = rows[1]
i_s, i_ex = H.index('Warp Stall Sampling (All Samples)'), H.index('Instructions Executed')
stall_cols = [k for k, h in enumerate(H) if h.startswith('stall_') and 'Not Issued' not in h]
data = []
for k, r in enumerate(rows[2:]):
    if len(r) <= i_s: continue
    s = float(r[i_s] or 0)
    top = sorted(((float(r[c] or 0), H[c]) for c in stall_cols), reverse=True)[:2]
    data.append((s, k, r[1].strip()[:70], r[i_ex], top))
tot = sum(d[0] for d in data) or 1
N = int(sys.argv[2]) if len(sys.argv) > 2 else 30
for s, k, src, ex, top in sorted(data, reverse=True)[:N]:
    print(f"{s/tot*100:5.1f}% #{k:5d} ex={ex:>10} {src:70s} {top[0][1]}={top[0][0]:.0f} {top[1][1]}={top[1][0]:.0f}")
