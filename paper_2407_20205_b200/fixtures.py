"""Seeded synthetic inputs for the BASELINE configs (host side, numpy).

No public dataset is involved: the paper's Monte Carlo trials are synthetic
too.  Every generator here is a counter-based splitmix64
stream, so any matrix of any family is reproducible from (seed, index):

* ``uniform_batch``  -- the reference's own trial stream (src/rng.py:49-71):
  matrix t of seed s is ``rng.sample_square(s, t, n)``; this is what
  ``montecarlo_zero`` draws, so batch results compare 1:1 with its tally.
* ``sparse_batch``   -- P(0) = 0.8, nonzeros uniform on {1, 2}.
* ``ones_batch``     -- all-ones (perm = n!, class 0 for n >= 3).
* ``perturbed_permutation_batch`` -- a random permutation matrix with one
  uniformly chosen entry set to a uniform class c; perm = c if the entry
  lies on the permutation, else 1 (closed form, ``perturbed_expected``).
* ``structured_batch`` -- config C3: the four families, count/4 each.

The sparse/permutation streams are new fixture code (the reference has no
such generator); their keys are documented below and recorded by bench.py.
"""

from __future__ import annotations

from typing import Tuple

import numpy as np

from . import rng

U64 = np.uint64
_GOLDEN = U64(rng.GOLDEN)
_MA = U64(0xBF58476D1CE4E5B9)
_MB = U64(0x94D049BB133111EB)

# family tags mixed into the per-matrix key: key = mix64(mix64(seed) ^ (tag << 40 | index + 1) * GOLDEN)
TAG_SPARSE = 1
TAG_PERM = 2


def _mix64(z: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = (z ^ (z >> U64(30))) * _MA
        z = (z ^ (z >> U64(27))) * _MB
        return z ^ (z >> U64(31))


def _stream(keys: np.ndarray, count: int) -> np.ndarray:
    """[len(keys), count] words of the splitmix64 streams starting at keys."""
    steps = (np.arange(1, count + 1, dtype=U64) * _GOLDEN)[None, :]
    with np.errstate(over="ignore"):
        return _mix64(keys[:, None] + steps)


def _keys(seed: int, tag: int, idx: np.ndarray) -> np.ndarray:
    s = _mix64(np.array([seed & rng.MASK64], dtype=U64))[0]
    with np.errstate(over="ignore"):
        return _mix64(s ^ ((U64(tag) << U64(40)) | (idx.astype(U64) + U64(1))) * _GOLDEN)


def uniform_batch(n: int, seed: int, t0: int, count: int) -> np.ndarray:
    """uint8 [count, n, n]: trials t0.. of the reference stream (classes)."""
    nn = n * n
    out = np.empty((count, nn), dtype=np.uint8)
    trials = np.arange(t0, t0 + count, dtype=np.int64)
    s = _mix64(np.array([seed & rng.MASK64], dtype=U64))[0]
    with np.errstate(over="ignore"):
        starts = _mix64(s ^ ((trials.astype(U64) + U64(1)) * _GOLDEN))
    words = max(4, (nn * 3) // 64 + 8)  # 32 slices/word, 3/4 accepted on average
    for lo in range(0, count, 4096):
        hi = min(count, lo + 4096)
        w = words
        while True:
            ws = _stream(starts[lo:hi], w)
            sl = ((ws[:, :, None] >> (U64(2) * np.arange(32, dtype=U64))[None, None, :]) & U64(3)).reshape(hi - lo, -1)
            ok = sl != U64(3)
            if (ok.sum(axis=1) >= nn).all():
                break
            w *= 2
        for k in range(hi - lo):
            out[lo + k] = sl[k][ok[k]][:nn].astype(np.uint8)
    return out.reshape(count, n, n)


def sparse_batch(n: int, seed: int, count: int, p_zero: float = 0.8) -> np.ndarray:
    """uint8 [count, n, n]; entry zero iff hi32(word) < p_zero * 2^32, else 1 + (word & 1)."""
    w = _stream(_keys(seed, TAG_SPARSE, np.arange(count)), n * n)
    thr = U64(int(p_zero * (1 << 32)))
    zero = (w >> U64(32)) < thr
    cls = (U64(1) + (w & U64(1))).astype(np.uint8)
    cls[zero] = 0
    return cls.reshape(count, n, n)


def ones_batch(n: int, count: int) -> np.ndarray:
    return np.ones((count, n, n), dtype=np.uint8)


def perturbed_permutation_batch(n: int, seed: int, count: int) -> Tuple[np.ndarray, np.ndarray]:
    """(uint8 [count, n, n], meta int64 [count, 4] = (i, j, c, on_perm)).

    Fisher-Yates with j = word % (k+1) for k = n-1..1, then position word % n^2
    and class word % 3 from the next two words of the same stream.
    """
    words = _stream(_keys(seed, TAG_PERM, np.arange(count)), n + 2)
    mats = np.zeros((count, n, n), dtype=np.uint8)
    meta = np.zeros((count, 4), dtype=np.int64)
    for b in range(count):
        sigma = list(range(n))
        for pos, k in enumerate(range(n - 1, 0, -1)):
            j = int(words[b, pos] % U64(k + 1))
            sigma[k], sigma[j] = sigma[j], sigma[k]
        mats[b, np.arange(n), sigma] = 1
        cell = int(words[b, n] % U64(n * n))
        c = int(words[b, n + 1] % U64(3))
        i, j = divmod(cell, n)
        mats[b, i, j] = c
        meta[b] = (i, j, c, int(sigma[i] == j))
    return mats, meta


def perturbed_expected(meta: np.ndarray) -> np.ndarray:
    """Closed-form class of each perturbed permutation matrix."""
    return np.where(meta[:, 3] == 1, meta[:, 2], 1).astype(np.int8)


def structured_batch(n: int, seed: int, count: int):
    """Config C3: [uniform | sparse | all-ones | perturbed permutation], count/4 each.

    Returns (entries uint8 [count, n, n], family int8 [count], expected int8
    [count] with -1 where no closed form exists (uniform, sparse)).
    """
    q = count // 4
    sizes = [q, q, q, count - 3 * q]
    uni = uniform_batch(n, seed, 0, sizes[0])
    spa = sparse_batch(n, seed, sizes[1])
    one = ones_batch(n, sizes[2])
    per, meta = perturbed_permutation_batch(n, seed, sizes[3])
    entries = np.concatenate([uni, spa, one, per])
    family = np.concatenate([np.full(s, f, dtype=np.int8) for f, s in enumerate(sizes)])
    fact_class = 0 if n >= 3 else (1 if n == 1 else 2)  # n! mod 3
    expected = np.concatenate([
        np.full(sizes[0], -1, dtype=np.int8),
        np.full(sizes[1], -1, dtype=np.int8),
        np.full(sizes[2], fact_class, dtype=np.int8),
        perturbed_expected(meta),
    ])
    return entries, family, expected
