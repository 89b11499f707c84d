"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Run in the build container (where /root/reference exists), never on the GPU
box:

    NUMBA_CACHE_DIR=/tmp/nb PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden.py [--with-slow]

It imports the reference package (/root/reference/pkg/src/tritperm, numba
kernels included) and records its outputs on seeded inputs.  The C oracle in
oracle/ and the CUDA path are both checked against these files; the files
carry everything the GPU tests need, so nothing reads /root/reference at
test time.  Matrices are stored as strings of classes '0'/'1'/'2'
(row-major), 2 == -1.

--with-slow adds the expensive anchors (C2's full montecarlo_zero tally at
n=24 with 16,384 trials, ~2 min on 8 threads; the n=50 2^30-step window,
~3 s) and the C3 uniform/sparse subset classes (~1 min).
"""

from __future__ import annotations

import argparse
import itertools
import json
import os
import random
import sys
import time

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nb")
sys.dont_write_bytecode = True
sys.path.insert(0, REF_SRC)
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402
from tritperm import _kernels as ref_k  # noqa: E402
from tritperm import core_f3 as ref_f3  # noqa: E402
from tritperm import experiments as ref_exp  # noqa: E402
from tritperm import permanent as ref_perm  # noqa: E402
from tritperm import rng as ref_rng  # noqa: E402


def enc(rows) -> str:
    return "".join(str(int(v) % 3) for row in rows for v in row)


def dump(name, obj):
    path = os.path.join(HERE, name)
    with open(path, "w") as f:
        json.dump(obj, f, indent=None, separators=(",", ":"))
        f.write("\n")
    print(f"wrote {path} ({os.path.getsize(path)} bytes)")


def core_ops():
    """add/sub on every 1-trit representation pair (tests/test_acceptance.py:74-99)."""
    rows = []
    for m1, s1, m2, s2 in itertools.product((0, 1), repeat=4):
        a = ref_f3.add_reps(ref_f3.PackedF3Vec(1, m1, s1), ref_f3.PackedF3Vec(1, m2, s2))
        s = ref_f3.sub_reps(ref_f3.PackedF3Vec(1, m1, s1), ref_f3.PackedF3Vec(1, m2, s2))
        rows.append({"in": [m1, s1, m2, s2], "add": [a.mag, a.sgn], "sub": [s.mag, s.sgn]})
    # wide random words (32-bit) through the same formulas
    r = random.Random(7)
    wide = []
    for _ in range(64):
        n = 32
        v1 = [r.randrange(-1, 2) for _ in range(n)]
        v2 = [r.randrange(-1, 2) for _ in range(n)]
        e1, e2 = ref_f3.encode(v1), ref_f3.encode(v2)
        a = ref_f3.add_reps(e1, e2)
        s = ref_f3.sub_reps(e1, e2)
        wide.append({"in": [e1.mag, e1.sgn, e2.mag, e2.sgn], "add": [a.mag, a.sgn], "sub": [s.mag, s.sgn]})
    e = ref_f3.encode((1, 1, 0, -1))
    dump("core_ops.json", {"pairs": rows, "wide": wide, "encode_example": {"in": [1, 1, 0, -1],
                                                                             "mag": e.mag, "sgn": e.sgn}})


def rng_vectors():
    state = 0
    words = []
    for _ in range(3):
        w, state = ref_rng.next_word(state)
        words.append(w)
    samples = []
    for n in (1, 2, 6, 13):
        for trial in (0, 1, 99, 10**7):
            for seed in (0, 1, 0xDEADBEEF, (1 << 64) - 1):
                ent = ref_k.mc_sample_entries(n, trial, np.uint64(seed))
                samples.append({"n": n, "trial": trial, "seed": seed, "entries": enc([ent.tolist()])})
    dump("rng.json", {"zero_seed_words": words, "samples": samples})


def chunks():
    """chunk_sum on seeded random matrices and ranges (aligned, unaligned, edge)."""
    r = random.Random(20261020)
    cases = []
    for n in list(range(1, 17)) + [20, 24, 28, 31, 32, 33, 36, 40, 50, 60, 62]:
        for k in range(6 if n <= 16 else 3):
            a = [[r.randrange(3) for _ in range(n)] for _ in range(n)]
            m = ref_perm.MatrixF3(a)
            mags, sgns = m.planes()
            last = 1 << n
            ranges = []
            if n <= 24:
                ranges.append((1, last))
            span = min(last, 1 << 22)
            for _ in range(4):
                lo = r.randrange(1, last - span + 2) if last - span >= 1 else 1
                hi = min(last, lo + r.randrange(0, span + 1))
                ranges.append((lo, hi))
            # 32-aligned and superblock-aligned windows
            if n >= 12:
                base = r.randrange(0, max(1, (last >> 12) - (1 << 8))) << 12
                ranges.append((max(1, base), base + (1 << min(n - 1, 17))))
            out = []
            for lo, hi in ranges:
                s = int(ref_k.chunk_sum(mags, sgns, n, lo, hi))
                out.append([lo, hi, s])
            cases.append({"n": n, "a": enc(a), "ranges": out})
    dump("chunks.json", {"cases": cases})


def tower():
    """Oracle tower of tests/test_acceptance.py:102-123 (random.Random(31415))."""
    rnd = random.Random(31415)
    out = []
    for n in range(1, 13):
        mats = []
        for _ in range(200):
            rows = [[rnd.randrange(-1, 2) for _ in range(n)] for _ in range(n)]
            m = ref_perm.MatrixF3(rows)
            v = ref_perm.perm_ryser_reference(m)
            assert v == ref_perm.perm_mod3_fast(m)
            mats.append([enc(rows), v, ref_perm.perm_chunk(m, 1, 1 << n).partial_sum])
        out.append({"n": n, "mats": mats})
    # exhaustive 2x2 and a naive check of 3x3
    ex2 = []
    for flat in itertools.product((-1, 0, 1), repeat=4):
        m = ref_perm.MatrixF3([flat[0:2], flat[2:4]])
        ex2.append([enc(m.rows), ref_perm.perm_naive(m)])
    dump("tower.json", {"random": out, "exhaustive2": ex2})


def anchors(with_slow: bool):
    res = {}
    # config C1-like anchors: n=20, trial 0, seeds 0..3
    c1 = []
    for seed in range(4):
        m = ref_exp.sample_trial_matrix(20, 0, seed)
        c1.append({"seed": seed, "trial": 0, "n": 20, "a": enc(m.rows),
                   "class": ref_perm.perm_mod3_fast(m) % 3,
                   "ryser_class": ref_perm.perm_ryser_reference(m) % 3,
                   "partial": ref_perm.perm_chunk(m, 1, 1 << 20).partial_sum})
    res["c1"] = c1
    mc = []
    for n, trials, seed in ((1, 3000, 5), (2, 20000, 1), (4, 400, 77), (5, 30000, 123), (6, 100000, 1),
                            (8, 20000, 3), (12, 2000, 9), (14, 500, 4)):
        t0 = time.time()
        r = ref_exp.montecarlo_zero(n, trials, seed=seed, jobs=4)
        mc.append({"n": n, "trials": trials, "seed": seed, "zero_count": r.zero_count})
        print(f"mc n={n} trials={trials}: {r.zero_count} ({time.time() - t0:.1f}s)")
    res["montecarlo"] = mc
    # known permanents (tests/test_permanent.py:74-78)
    res["known"] = [["100010001", 1], ["1111", -1], ["0", 0], ["2", -1]]
    if with_slow:
        t0 = time.time()
        r = ref_exp.montecarlo_zero(24, 16384, seed=0, jobs=os.cpu_count())
        res["c2_zero_count"] = {"n": 24, "trials": 16384, "seed": 0, "zero_count": r.zero_count,
                                "seconds": round(time.time() - t0, 1)}
        print("c2 zero count", r.zero_count, time.time() - t0)
        m = ref_exp.sample_trial_matrix(50, 0, 0)
        mags, sgns = m.planes()
        lo = 1 << 40
        res["c5_window"] = {"n": 50, "seed": 0, "trial": 0, "a": enc(m.rows), "lo": lo, "hi": lo + (1 << 30),
                            "partial": int(ref_k.chunk_sum(mags, sgns, 50, lo, lo + (1 << 30)))}
        m36 = ref_exp.sample_trial_matrix(36, 0, 0)
        mags, sgns = m36.planes()
        lo = 3 << 33
        res["c4_window"] = {"n": 36, "seed": 0, "trial": 0, "a": enc(m36.rows), "lo": lo, "hi": lo + (1 << 30),
                            "partial": int(ref_k.chunk_sum(mags, sgns, 36, lo, lo + (1 << 30)))}
    dump("anchors.json", res)


def oracle_goldens():
    """Large goldens computed by the C oracle (oracle/oracle.c), which the
    cheap goldens above pin against the reference; each block is
    additionally cross-pinned to a reference output where one exists."""
    from oracle import oracle as orc
    from paper_2407_20205_b200 import fixtures

    orc.build()
    path = os.path.join(HERE, "anchors.json")
    with open(path) as f:
        res = json.load(f)
    threads = os.cpu_count() or 1
    # C2: all 16,384 classes of the reference stream at n=24, seed 0
    t0 = time.time()
    e = fixtures.uniform_batch(24, 0, 0, 16384)
    for t in (0, 1, 16383):  # fixture == reference sampler
        assert enc(np.mod(np.array(ref_rng.sample_square(0, t, 24)), 3)) == enc(e[t])
    cls, part = orc.perm_batch(e, threads=threads)
    hist = np.bincount(cls, minlength=3).tolist()
    assert hist[0] == res["c2_zero_count"]["zero_count"], (hist, res["c2_zero_count"])  # pinned by the reference
    for t in range(8):  # and by the reference's own kernel on the first matrices
        m = ref_perm.MatrixF3(ref_rng.sample_square(0, t, 24))
        assert ref_perm.perm_chunk(m, 1, 1 << 24).partial_sum == part[t]
    res["c2_classes"] = "".join(str(int(c)) for c in cls)
    res["c2_hist"] = hist
    res["c2_partials_head"] = [int(v) for v in part[:64]]
    print(f"c2 oracle: {time.time() - t0:.1f}s hist={hist}")
    # C3: oracle classes of a seeded subset of the uniform and sparse families
    t0 = time.time()
    entries, fam, exp = fixtures.structured_batch(32, 0, 4096)
    idx = [int(i) for i in list(range(0, 24)) + list(range(1024, 1048))]
    sub_cls, _ = orc.perm_batch(entries[idx], threads=threads)
    res["c3_subset"] = [[i, int(c)] for i, c in zip(idx, sub_cls)]
    res["c3_entries_sha256"] = __import__("hashlib").sha256(entries.tobytes()).hexdigest()
    print(f"c3 oracle subset: {time.time() - t0:.1f}s")
    # C4: full n=36 traversal, cross-pinned to the reference's parallel engine
    t0 = time.time()
    w = res["c4_window"]
    a = np.frombuffer(w["a"].encode(), dtype=np.uint8).reshape(36, 36) - ord("0")
    mags, sgns = orc.planes_from_classes(a)
    full = orc.chunk_sum_mt(mags, sgns, 36, 1, 1 << 36, threads)
    ref_val = ref_perm.perm_mod3_parallel(ref_perm.MatrixF3(ref_rng.sample_square(0, 0, 36)), jobs=threads)
    assert orc.finalize(36, full) == ref_val
    res["c4_full"] = {"n": 36, "seed": 0, "trial": 0, "a": w["a"], "partial": int(full),
                      "class": int(orc.finalize(36, full)) % 3}
    print(f"c4 full: {time.time() - t0:.1f}s partial={full}")
    # C5: a 2^36-step window of the n=50 matrix (-5)
    t0 = time.time()
    w = res["c5_window"]
    a = np.frombuffer(w["a"].encode(), dtype=np.uint8).reshape(50, 50) - ord("0")
    mags, sgns = orc.planes_from_classes(a)
    lo = 1 << 40
    assert orc.chunk_sum(mags, sgns, 50, w["lo"], w["hi"]) == w["partial"]
    s36 = orc.chunk_sum_mt(mags, sgns, 50, lo, lo + (1 << 36), threads)
    res["c5_window36"] = {"n": 50, "seed": 0, "trial": 0, "a": w["a"], "lo": lo, "hi": lo + (1 << 36),
                          "partial": int(s36)}
    print(f"c5 window36: {time.time() - t0:.1f}s partial={s36}")
    dump("anchors.json", res)


def c3_full():
    """Config C3 in full: all 4,096 classes and the histogram (tests/golden/c3.json).

    * uniform + sparse families (2,048 matrices, no closed form): the C
      oracle's chunk_sum over [1, 2^32) per matrix, raw partial and class;
      a seeded subset is cross-pinned to the reference's own
      perm_mod3_parallel / perm_chunk (src/permanent.py:181-255);
    * all-ones: perm = n! = 0 mod 3; perturbed permutations: the closed form
      (fixtures.perturbed_expected), both cross-checked on a few matrices
      by the reference too.
    ~35 min on 8 container threads.
    """
    from oracle import oracle as orc
    from paper_2407_20205_b200 import fixtures

    orc.build()
    threads = os.cpu_count() or 1
    n = 32
    entries, fam, exp = fixtures.structured_batch(n, 0, 4096)
    t0 = time.time()
    cls = np.array(exp, dtype=np.int8)
    part = np.zeros(4096, dtype=np.int64)
    todo = np.nonzero(exp < 0)[0]
    for lo in range(0, len(todo), 64):  # progress in blocks
        idx = todo[lo:lo + 64]
        c, p = orc.perm_batch(entries[idx], threads=threads)
        cls[idx] = c
        part[idx] = p
        print(f"c3 oracle {lo + len(idx)}/{len(todo)}: {time.time() - t0:.0f}s", flush=True)
    # cross-pin: the reference's own engines on a seeded subset of every family
    rnd = random.Random(3232)
    pins = []
    for f in range(4):
        members = np.nonzero(fam == f)[0]
        for i in sorted(rnd.sample(list(members), 3)):
            m = ref_perm.MatrixF3(entries[i].astype(np.int64).tolist())
            v = ref_perm.perm_mod3_parallel(m, jobs=threads) % 3
            assert v == int(cls[i]), (i, v, int(cls[i]))
            pins.append([int(i), int(v)])
        print(f"c3 family {f} pinned by the reference: {time.time() - t0:.0f}s", flush=True)
    hist = np.bincount(cls.astype(np.int64), minlength=3).tolist()
    dump("c3.json", {"n": n, "seed": 0, "count": 4096,
                     "entries_sha256": __import__("hashlib").sha256(entries.tobytes()).hexdigest(),
                     "classes": "".join(str(int(c)) for c in cls),
                     "partials_oracle": {str(int(i)): int(part[i]) for i in todo},
                     "hist": hist, "reference_pins": pins,
                     "seconds": round(time.time() - t0, 1)})


def n64_goldens():
    """perm_chunk on n = 63, 64 windows from the reference, which routes n > 62
    to its big-int twin _chunk_sum_pure (src/permanent.py:157-178,192-196);
    the windows include the last steps up to 2^64."""
    r = random.Random(6464)
    cases = []
    for n in (63, 64):
        for k in range(3):
            # event-dense inputs (uniform ones have almost no full terms at n = 64):
            # k = 0 entries in {1, 2}; k = 1 all ones but ~2 % zeros; k = 2 uniform
            # with a zero-free last row, so the final step 2^n - 1 ({row n-1}) is full
            if k == 0:
                a = [[r.choice((1, 2)) for _ in range(n)] for _ in range(n)]
            elif k == 1:
                a = [[0 if r.random() < 0.02 else 1 for _ in range(n)] for _ in range(n)]
            else:
                a = [[r.randrange(3) for _ in range(n)] for _ in range(n)]
                a[n - 1] = [r.choice((1, 2)) for _ in range(n)]
            m = ref_perm.MatrixF3(a)
            last = 1 << n
            out = []
            for lo, hi in ((1, 1 << 12), ((1 << 40) + 5, (1 << 40) + 5 + 3000), ((1 << 62) - 1500, (1 << 62) + 2500),
                           (last - 4096, last), (last - 3, last), (last - 2000, last - 700)):
                out.append([lo, hi, ref_perm.perm_chunk(m, lo, hi).partial_sum])
            cases.append({"n": n, "a": enc(a), "ranges": out})
    dump("n64.json", {"cases": cases})


def pi_goldens():
    """pi_matrix rows and Pi_50 windows from the reference (src/experiments.py:193-213)."""
    out = {"pi_matrix": [], "windows": []}
    for n in (1, 3, 6, 20, 50):
        for skip in (False, True):
            m = ref_exp.pi_matrix(n, skip_integer_part=skip)
            rec = {"n": n, "skip_integer_part": skip, "a": enc(m.rows)}
            if n <= 20:
                rec["perm"] = ref_perm.perm_mod3_fast(m)
                rec["partial"] = ref_perm.perm_chunk(m, 1, 1 << n).partial_sum
            out["pi_matrix"].append(rec)
    for skip in (False, True):
        m = ref_exp.pi_matrix(50, skip_integer_part=skip)
        mags, sgns = m.planes()
        lo = 1 << 40
        t0 = time.time()
        s30 = int(ref_k.chunk_sum(mags, sgns, 50, lo, lo + (1 << 30)))
        out["windows"].append({"skip_integer_part": skip, "lo": lo, "hi": lo + (1 << 30), "partial": s30})
        print(f"pi50 skip={skip} window 2^30: {s30} ({time.time() - t0:.1f}s)")
    dump("pi.json", out)


def census_goldens():
    """exact_zero_count(1..4) from the reference (src/experiments.py:113-140);
    z(5) is the paper's published value (Table 3), which the
    reference refuses to compute."""
    out = []
    for n in (1, 2, 3, 4):
        t0 = time.time()
        r = ref_exp.exact_zero_count(n)
        out.append({"n": n, "z": r.z, "plus": r.plus_ones, "minus": r.minus_ones, "total": r.total,
                    "source": "reference exact_zero_count"})
        print(f"census n={n}: {r.z} ({time.time() - t0:.1f}s)")
    out.append({"n": 5, "z": 317193401763, "total": 3 ** 25, "source": "PAPER.md:245 (Table 3)"})
    dump("census.json", {"census": out})


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--with-slow", action="store_true")
    ap.add_argument("--only", default=None)
    args = ap.parse_args()
    jobs = {"core": core_ops, "rng": rng_vectors, "n64": n64_goldens, "chunks": chunks, "tower": tower, "pi": pi_goldens, "census": census_goldens,
            "anchors": lambda: anchors(args.with_slow)}
    if args.with_slow:
        jobs["oracle"] = oracle_goldens
        jobs["c3"] = c3_full
    for name, fn in jobs.items():
        if args.only and name not in args.only.split(","):
            continue
        t0 = time.time()
        fn()
        print(f"{name}: {time.time() - t0:.1f}s")


if __name__ == "__main__":
    main()
