"""Time the C3 workload (4,096 x 32x32 structured, bench.py's seed) per family
through perm_mod3_batch: where the C3 step goes.  Prints one JSON line per
family: wall ms per call (after a warm-up, device-synchronised), terms/s, and
the fraction of pairs the bucketed walk tested."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2407_20205_b200 as tp  # noqa: E402
from paper_2407_20205_b200 import _kernels, fixtures  # noqa: E402

NAMES = ["uniform", "sparse", "all-ones", "perturbed permutation"]


def main():
    n = 32
    entries, family, _ = fixtures.structured_batch(n, 0, 4096)
    for f in range(4):
        e = np.ascontiguousarray(entries[family == f])
        tp.perm_mod3_batch(e, device=0)  # warm-up
        _kernels.walk_tested(0)
        reps = 3
        t0 = time.perf_counter()
        for _ in range(reps):
            tp.perm_mod3_batch(e, device=0)
        ms = (time.perf_counter() - t0) * 1e3 / reps
        tested = _kernels.walk_tested(0) / reps
        terms = len(e) * 2.0 ** n
        print(json.dumps({"family": NAMES[f], "matrices": int(len(e)), "ms": ms, "terms_per_s": terms / (ms * 1e-3),
                          "tested_pairs_frac": tested / terms}))


if __name__ == "__main__":
    main()
