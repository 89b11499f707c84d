"""Exact census z(n) = #{A in F3^{n x n} : perm(A) = 0 mod 3} on the GPU
(SURVEY next-2).  z(1..4) match the reference's exact_zero_count, z(5) the
paper's Table 3; n = 6 is beyond the paper.

    python tools/census.py [--n 1,2,3,4,5,6]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_20205_b200 as tp  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", default="1,2,3,4,5,6")
args = ap.parse_args()
for n in [int(x) for x in args.n.split(",")]:
    t0 = time.perf_counter()
    r = tp.exact_zero_count(n)
    dt = time.perf_counter() - t0
    print(json.dumps({"n": n, "z": r.z, "plus_ones": r.plus_ones, "minus_ones": r.minus_ones, "total": r.total,
                      "ratio": r.ratio, "seconds": round(dt, 3)}), flush=True)
