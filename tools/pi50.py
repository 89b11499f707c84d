"""perm(Pi_50) mod 3 on the GPU (SURVEY next-3; PAPER.md:226 reports -1).

Runs the full 2^50-subset traversal of pi_matrix(50) for both readings of
Pi_n (digits from the leading "3", or from the first fractional digit,
SPEC.md:415) and prints one JSON record per variant.

    python tools/pi50.py [--variants 0,1]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_20205_b200 as tp  # noqa: E402
from paper_2407_20205_b200 import _kernels  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--variants", default="0,1")
args = ap.parse_args()
for v in [int(x) for x in args.variants.split(",")]:
    m = tp.pi_matrix(50, skip_integer_part=bool(v))
    mags, sgns = m.planes()
    t0 = time.perf_counter()
    p, q = _kernels.chunk_counts(mags, sgns, 50, 1, 1 << 50)
    dt = time.perf_counter() - t0
    s = p - q
    perm = tp.cmod3(-s if 50 & 1 else s)
    print(json.dumps({"matrix": "pi_matrix(50, skip_integer_part=%s)" % bool(v), "plus": p, "minus": q,
                      "partial_sum": s, "perm_mod3": perm, "seconds": round(dt, 2),
                      "terms_per_s": (1 << 50) / dt, "device": _kernels.device_info()}), flush=True)
