"""A small run of every walk kernel family for compute-sanitizer (memcheck,
racecheck, synccheck, initcheck), checked against the C oracle.  No torch:
the library, numpy and the oracle only, so the sanitizer sees our kernels.

    compute-sanitizer --tool racecheck python tools/sanitize_case.py

Cases: a bucketed 2-key batch (n = 24), a 3-key batch (n = 28), a weighted
(deduplicated) all-ones matrix, ranges with generic heads and tails on the
3-key walk at n = 32 and the wide walk at n = 34, 36, the packed / lane walks
(n = 16, 20) and the thread-per-matrix kernel (n = 9)."""
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import numpy as np  # noqa: E402

from oracle import oracle  # noqa: E402
from paper_2407_20205_b200 import _kernels, fixtures  # noqa: E402

oracle.build()
threads = os.cpu_count() or 4
for n, B, seed in ((24, 8, 1), (28, 2, 2), (16, 40, 5), (20, 3, 6), (9, 64, 7)):
    e = fixtures.uniform_batch(n, seed, 0, B)
    cls, part, hist = _kernels.perm_batch(e)
    want_cls, want_part = oracle.perm_batch(e, threads=threads)
    assert np.array_equal(part, want_part), (n, "partials")
    assert np.array_equal(cls, want_cls), (n, "classes")
    print(f"n={n} B={B}: ok", flush=True)
ones = np.ones((2, 26, 26), np.uint8)
cls, part, hist = _kernels.perm_batch(ones)
mags, sgns = oracle.planes_from_classes(ones[0])
assert part[0] == part[1] == oracle.chunk_sum_mt(mags, sgns, 26, 1, 1 << 26, threads), "all-ones (weighted)"
print("all-ones n=26 (weighted walk): ok", flush=True)
for n in (32, 34, 36):
    a = fixtures.uniform_batch(n, 8, 0, 1)[0]
    mags, sgns = oracle.planes_from_classes(a)
    lo, hi = (5 << 26) + 12345, (5 << 26) + (1 << 27) + 999
    assert _kernels.chunk_sum(mags, sgns, n, lo, hi) == oracle.chunk_sum_mt(mags, sgns, n, lo, hi, threads), n
    print(f"n={n} range (bucketed middle + generic head/tail): ok", flush=True)
print("sanitize case ok")
