"""Monte Carlo zero-permanent study on the B200 (reference: src/experiments.py).

``montecarlo_zero`` keeps the reference signature and result type: trial t's
matrix depends only on (seed, t) (splitmix64 stream, ``rng``), so the tally
is bit-identical to the reference's for the same (n, trials, seed), and
independent of ``jobs``.  Sampling, traversal and tallying all run on the
device (tp_mc_zero_count: k_sample -> k_walk_* -> k_finalize).

Added: ``montecarlo_hist`` (counts of perm = 0, +1, -1) and ``trial_classes``
(per-trial classes), which the reference does not expose.
"""

from __future__ import annotations

from dataclasses import dataclass
from math import sqrt

import numpy as np

from . import _kernels, rng
from .permanent import MAX_N, MatrixF3, resolve_jobs

MC_MAX_N = 63  # the reference's guard (src/experiments.py:39); the kernels go to MAX_N
EXACT_MAX_N = 6  # the reference stops at 4 (src/experiments.py:37)


@dataclass(frozen=True)
class ExactCountResult:
    """Exact census of perm mod 3 over all n x n trit matrices (src/experiments.py:41-60)."""

    n: int
    z: int
    plus_ones: int
    minus_ones: int
    total: int

    @property
    def ratio(self) -> float:
        return self.z / self.total


def exact_zero_count(n: int) -> ExactCountResult:
    """Census of permanent values over all 3**(n*n) matrices, n <= 6, on the GPU
    (tp_exact_census; the reference enumerates and refuses n > 4)."""
    if n < 1:
        raise ValueError("n must be >= 1")
    if n > EXACT_MAX_N:
        raise ValueError(f"exact census supports n <= {EXACT_MAX_N} (3**{(n - 2) * n} rank computations)")
    z, p, m = _kernels.exact_census(n)
    return ExactCountResult(n=n, z=z, plus_ones=p, minus_ones=m, total=3 ** (n * n))


@dataclass(frozen=True)
class McResult:
    """Tally of one Monte Carlo run; (n, trials, seed) fixes zero_count."""

    n: int
    trials: int
    zero_count: int
    seed: int

    @property
    def p_hat(self) -> float:
        return self.zero_count / self.trials

    @property
    def stderr(self) -> float:
        p = self.p_hat
        return sqrt(p * (1.0 - p) / self.trials)


@dataclass(frozen=True)
class McHistogram:
    """Counts of perm mod 3 = 0, +1, -1 over trials [0, trials)."""

    n: int
    trials: int
    seed: int
    zeros: int
    plus_ones: int
    minus_ones: int


def sample_trial_matrix(n: int, trial: int, seed: int) -> MatrixF3:
    """The exact matrix ``montecarlo_zero`` evaluates as `trial`."""
    return MatrixF3(rng.sample_square(seed & rng.MASK64, trial, n))


def _validate(n: int, trials: int, max_n: int) -> None:
    if n < 1:
        raise ValueError("n must be >= 1")
    if n > max_n:
        raise ValueError(f"montecarlo_zero is limited to n <= {max_n}")
    if trials < 1:
        raise ValueError("trials must be >= 1")


def montecarlo_zero(n: int, trials: int, seed: int = 0, jobs=None) -> McResult:
    """Zero-permanent frequency over uniform random trit matrices."""
    _validate(n, trials, MC_MAX_N)
    resolve_jobs(jobs)  # same validation as the reference; the GPU ignores the count
    seed64 = seed & rng.MASK64
    zeros = _kernels.mc_zero_count(n, 0, trials, seed64)
    return McResult(n=n, trials=trials, zero_count=zeros, seed=seed64)


def montecarlo_hist(n: int, trials: int, seed: int = 0) -> McHistogram:
    """Counts of perm = 0, +1, -1 over the same trials as ``montecarlo_zero``."""
    _validate(n, trials, MAX_N)
    seed64 = seed & rng.MASK64
    h = _kernels.mc_hist(n, 0, trials, seed64)
    return McHistogram(n=n, trials=trials, seed=seed64, zeros=int(h[0]), plus_ones=int(h[1]),
                       minus_ones=int(h[2]))


def trial_classes(n: int, t0: int, count: int, seed: int = 0) -> np.ndarray:
    """int8 classes {0, 1, 2} of perm mod 3 for trials [t0, t0+count)."""
    _validate(n, max(count, 1), MAX_N)
    return _kernels.mc_classes(n, t0, count, seed & rng.MASK64)
