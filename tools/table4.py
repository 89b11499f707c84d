"""The paper's Monte Carlo study (Table 4: n = 6..30, 10^11
down to 10^6 trials; "about one full day on 128 processors") on one B200,
through the reference-facing API ``montecarlo_zero`` (device sampler + walk
+ finalize + histogram, DESIGN.md sections 1-5).

The trial stream is the reference's splitmix64 stream with seed 0, not the
paper's (unpublished) generator, so the tallies are a second, independent
sample: each row reports the z-score of the difference of the two zero
frequencies, (p_here - p_paper) / sqrt(p (1 - p) (1/N_here + 1/N_paper)).

    python tools/table4.py [--scale 1.0] [--nmin 6] [--nmax 30] [--seed 0]

One JSON record per n, then a summary record."""
import argparse
import json
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_20205_b200 as tp  # noqa: E402
from paper_2407_20205_b200 import _kernels  # noqa: E402

# n: (zero count, log10 trials)
PAPER = {6: (35456365448, 11), 7: (34209345718, 11), 8: (33623043873, 11), 9: (33417515901, 11),
         10: (33358878343, 11), 11: (3334206857, 10), 12: (3333537904, 10), 13: (3333483177, 10),
         14: (3333394825, 10), 15: (333332350, 9), 16: (333308622, 9), 17: (333314098, 9),
         18: (33331991, 8), 19: (33338438, 8), 20: (33338902, 8), 21: (3332782, 7), 22: (3333672, 7),
         23: (3336968, 7), 24: (3333518, 7), 25: (3332961, 7), 26: (3335524, 7), 27: (3332955, 7),
         28: (333743, 6), 29: (334097, 6), 30: (333080, 6)}

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=float, default=1.0, help="fraction of the paper's trial counts")
ap.add_argument("--nmin", type=int, default=6)
ap.add_argument("--nmax", type=int, default=30)
ap.add_argument("--seed", type=int, default=0)
args = ap.parse_args()

tot_s = tot_terms = 0.0
worst = 0.0
for n in range(args.nmin, args.nmax + 1):
    zp, lg = PAPER[n]
    n_paper = 10 ** lg
    trials = max(1, int(round(n_paper * args.scale)))
    t0 = time.perf_counter()
    r = tp.montecarlo_zero(n, trials, seed=args.seed)
    dt = time.perf_counter() - t0
    p_here, p_paper = r.zero_count / trials, zp / n_paper
    p = (r.zero_count + zp) / (trials + n_paper)
    z = (p_here - p_paper) / math.sqrt(p * (1 - p) * (1 / trials + 1 / n_paper))
    kernel, _ = _kernels.walk_info(n, min(trials, 1 << 16))
    tot_s += dt
    tot_terms += trials * float(1 << n)
    worst = max(worst, abs(z))
    print(json.dumps({"n": n, "trials": trials, "zero_count": r.zero_count, "zero_fraction": p_here,
                      "paper_zero_count": zp, "paper_trials": n_paper, "paper_zero_fraction": p_paper,
                      "z_vs_paper": round(z, 3), "seconds": round(dt, 3), "trials_per_s": trials / dt,
                      "terms_per_s": trials * float(1 << n) / dt, "kernel": kernel, "seed": args.seed}), flush=True)
print(json.dumps({"summary": "Table 4, n = %d..%d at %.3g x the paper's trial counts" % (args.nmin, args.nmax, args.scale),
                  "seconds": round(tot_s, 1), "terms": tot_terms, "terms_per_s": tot_terms / tot_s,
                  "max_abs_z_vs_paper": round(worst, 3), "device": _kernels.device_info()}), flush=True)
