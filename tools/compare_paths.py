"""Time the C2 workload (16,384 x 24x24, reference trial stream, seed 0)
through perm_mod3_batch on every exact path -- the bucketed walk (the
default, TRITPERM_BUCKET=1; =2 with unpacked pair tests), the packed walk
(TRITPERM_BUCKET=0) and the tcgen05 pair test (TRITPERM_TC=1) -- and check
that they return the same classes and raw partials.  Host-timed (H2D, pack, walk, finalize, D2H): the numbers quoted in
DESIGN.md sections 5b and 5c.

    python tools/compare_paths.py [--batch 16384] [--n 24] [--reps 3]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2407_20205_b200 as tp  # noqa: E402
from paper_2407_20205_b200 import fixtures  # noqa: E402

PATHS = {
    "packed walk": {"TRITPERM_BUCKET": "0", "TRITPERM_TC": "0"},
    "bucketed (default)": {"TRITPERM_BUCKET": "1", "TRITPERM_TC": "0"},
    "bucketed, pair tests": {"TRITPERM_BUCKET": "2", "TRITPERM_TC": "0"},
    "tcgen05 pair test": {"TRITPERM_BUCKET": "0", "TRITPERM_TC": "1"},
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=16384)
    ap.add_argument("--n", type=int, default=24)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    e = fixtures.uniform_batch(a.n, 0, 0, a.batch)
    ref = None
    for name, env in PATHS.items():
        os.environ.update(env)
        tp.perm_mod3_batch(e[:64], device=0)  # warm-up (module load, workspaces)
        best = float("inf")
        for _ in range(a.reps):
            t0 = time.perf_counter()
            cls, part, hist = tp.perm_mod3_batch(e, device=0)
            best = min(best, time.perf_counter() - t0)
        same = ref is None or (np.array_equal(cls, ref[0]) and np.array_equal(part, ref[1]))
        if ref is None:
            ref = (cls, part)
        print(f"{name:26s} {best * 1e3:8.1f} ms  {a.batch * 2.0 ** a.n / best:.3e} terms/s  "
              f"hist {hist.tolist()}  {'same' if same else 'MISMATCH'}")


if __name__ == "__main__":
    main()
