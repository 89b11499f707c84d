"""Permanent engines over GF(3), B200 edition.

Same public surface as the reference module (src/permanent.py): ``MatrixF3``,
``ChunkResult``, ``cmod3``, ``perm_chunk``, ``perm_mod3_fast``,
``perm_mod3_parallel``, ``split_steps``, ``resolve_jobs``; values returned
centred in {-1, 0, 1}, validation errors raised as ValueError before any
device work, results invariant to ``jobs``.  Every traversal runs in the
sm_100a kernels behind ``_kernels`` (no CPU engine, no fallback).

Added for the batched study: ``perm_mod3_batch`` (per-matrix classes and the
histogram of a uint8 [B, n, n] batch in one launch sequence).

Differences from the reference, by design:
* ``jobs`` in ``perm_mod3_parallel`` is the number of GPUs the range is
  split across (capped by the visible device count, env ``TRITPERM_GPUS``);
  under ``torch.distributed`` with world_size > 1 the range is split across
  ranks instead and joined by one NCCL all-reduce (``parallel.py``).
* the naive / unpacked engines (``perm_naive``, ``perm_ryser_reference``)
  are CPU oracles and live in ``oracle/`` with the tests, not here.
"""

from __future__ import annotations

import os
from dataclasses import dataclass
from typing import Iterable, List, Tuple

import numpy as np

from . import _kernels
from .core_f3 import PackedF3Vec, encode

# Largest n whose planes fit one uint64 and whose step range fits the range
# ABI (hi <= 2^63); full traversals go up to MAX_N through the batch ABI.
SINGLE_LIMB_MAX_N = 63
MAX_N = 64

ENV_THREADS = "TRITPERM_THREADS"
ENV_GPUS = "TRITPERM_GPUS"


def cmod3(k: int) -> int:
    """Centred residue of k modulo 3: one of -1, 0, 1."""
    r = k % 3
    return -1 if r == 2 else r


class MatrixF3:
    """Square matrix over GF(3), normalised to centred entries.

    Accepts any integer entries and reduces them mod 3 ({0,1,2} and
    {-1,0,1} describe the same matrix); keeps the packed rows the kernels
    consume.
    """

    __slots__ = ("n", "rows", "packed_rows")

    def __init__(self, rows: Iterable[Iterable[int]]):
        centred = tuple(tuple(cmod3(int(v)) for v in row) for row in rows)
        n = len(centred)
        if n == 0:
            raise ValueError("matrix must have at least one row")
        for row in centred:
            if len(row) != n:
                raise ValueError(f"matrix must be square, got a row of length {len(row)} for n={n}")
        self.n = n
        self.rows = centred
        self.packed_rows: Tuple[PackedF3Vec, ...] = tuple(encode(r) for r in centred)

    def __eq__(self, other) -> bool:
        return isinstance(other, MatrixF3) and self.rows == other.rows

    def __hash__(self) -> int:
        return hash(self.rows)

    def __repr__(self) -> str:
        return f"MatrixF3({[list(r) for r in self.rows]!r})"

    def to_numpy(self) -> np.ndarray:
        """Centred entries as int64."""
        return np.array(self.rows, dtype=np.int64)

    def classes(self) -> np.ndarray:
        """Entries as uint8 classes {0, 1, 2} (2 == -1)."""
        return np.mod(self.to_numpy(), 3).astype(np.uint8)

    def planes(self) -> Tuple[np.ndarray, np.ndarray]:
        """Per-row (mag, sgn) planes as uint64 arrays (row t -> word t)."""
        if self.n > MAX_N:
            raise ValueError(f"packed planes only fit uint64 for n <= {MAX_N}")
        mags = np.array([r.mag for r in self.packed_rows], dtype=np.uint64)
        sgns = np.array([r.sgn for r in self.packed_rows], dtype=np.uint64)
        return mags, sgns


@dataclass(frozen=True)
class ChunkResult:
    """Partial sum over traversal steps lo..hi-1 (half-open, 1-based)."""

    lo: int
    hi: int
    partial_sum: int


def _as_matrix(m) -> MatrixF3:
    return m if isinstance(m, MatrixF3) else MatrixF3(m)


def _finalize(n: int, s: int) -> int:
    return cmod3(-s if n & 1 else s)


def _check_n(n: int) -> None:
    if n > MAX_N:
        raise ValueError(f"the B200 engines support n <= {MAX_N}, got n={n}")


def perm_chunk(m, lo: int, hi: int) -> ChunkResult:
    """Partial sum of the packed traversal over steps lo..hi-1.

    Steps are 1-based and half-open, the full job is (1, 2**n); partial sums
    of adjacent ranges add exactly.  Runs ``tp_range_sum`` on one device
    (n = 64: ``tp_range_sum_ex``, whose end may be 2**64; the reference's
    big-int twin covers the same case, src/permanent.py:157-178,192-196).
    """
    m = _as_matrix(m)
    last = 1 << m.n
    if not 1 <= lo <= hi <= last:
        raise ValueError(f"need 1 <= lo <= hi <= 2**n, got lo={lo} hi={hi} n={m.n}")
    _check_n(m.n)
    mags, sgns = m.planes()
    return ChunkResult(lo=lo, hi=hi, partial_sum=_kernels.chunk_sum(mags, sgns, m.n, lo, hi))


def perm_mod3_fast(m) -> int:
    """Permanent mod 3 (centred) of one matrix on one GPU."""
    m = _as_matrix(m)
    _check_n(m.n)
    if m.n <= SINGLE_LIMB_MAX_N:
        return _finalize(m.n, perm_chunk(m, 1, 1 << m.n).partial_sum)
    cls, _, _ = _kernels.perm_batch(m.classes()[None], partials=False)
    return cmod3(int(cls[0]))


def resolve_jobs(jobs=None) -> int:
    """Worker count: explicit argument, else TRITPERM_THREADS, else CPUs."""
    if jobs is None:
        env = os.environ.get(ENV_THREADS)
        jobs = int(env) if env is not None else (os.cpu_count() or 1)
    jobs = int(jobs)
    if jobs < 1:
        raise ValueError(f"jobs must be >= 1, got {jobs}")
    return jobs


def split_steps(n: int, jobs: int) -> List[Tuple[int, int]]:
    """Partition steps 1..2**n-1 into `jobs` contiguous ranges (empty kept)."""
    total = (1 << n) - 1
    edges = [1 + (total * k) // jobs for k in range(jobs + 1)]
    return [(edges[k], edges[k + 1]) for k in range(jobs)]


def resolve_gpus(jobs=None) -> List[int]:
    """Devices used by ``perm_mod3_parallel``: min(jobs, $TRITPERM_GPUS, visible)."""
    visible = _kernels.device_count()
    if visible < 1:
        raise RuntimeError("no B200 (sm_100) device visible: the B200 engines have no CPU fallback")
    cap = visible
    env = os.environ.get(ENV_GPUS)
    if env is not None:
        cap = max(1, min(cap, int(env)))
    return list(range(min(resolve_jobs(jobs), cap)))


def perm_mod3_parallel(m, jobs=None) -> int:
    """Permanent mod 3 with the traversal split across GPUs.

    Every part is an exact integer and addition the only combination step,
    so the answer is identical for every ``jobs``.  Under torch.distributed
    (world_size > 1) each rank takes one ``split_steps`` part and the counters
    meet in one NCCL all-reduce.
    """
    m = _as_matrix(m)
    _check_n(m.n)
    from . import parallel

    if parallel.world_size() > 1:
        return parallel.perm_mod3_distributed(m)
    devices = resolve_gpus(jobs)
    if m.n > SINGLE_LIMB_MAX_N or len(devices) == 1:
        return perm_mod3_fast(m)
    mags, sgns = m.planes()
    p, q = _kernels.chunk_counts_multi(mags, sgns, m.n, 1, 1 << m.n, devices)
    return _finalize(m.n, p - q)


def perm_mod3_batch(entries, device=None):
    """Per-matrix perm mod 3 of a batch.

    ``entries``: uint8-compatible array [B, n, n] (values reduced mod 3) or a
    sequence of matrices.  Returns (classes int8[B] in {0, 1, 2},
    partials int64[B] of the raw Gray sums (n <= 62, else None),
    hist int64[3] counts of classes 0, 1, 2).
    """
    arr = np.asarray(entries)
    if arr.ndim != 3 or arr.shape[1] != arr.shape[2]:
        raise ValueError("entries must have shape [B, n, n]")
    if arr.shape[1] < 1:
        raise ValueError("matrix must have at least one row")
    _check_n(arr.shape[1])
    if arr.dtype != np.uint8:
        arr = np.mod(arr.astype(np.int64), 3).astype(np.uint8)
    return _kernels.perm_batch(arr, device=device)
