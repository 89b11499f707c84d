"""Checkpoint / resume of one long traversal (the n = 50 class of runs).

The reference has no checkpointing; its natural unit is ``ChunkResult``
(src/permanent.py:103-109): partial sums of adjacent step ranges add exactly
 and a range is a pure function of (rows, lo, hi)
(src/_kernels.py:96-97), so a run can be cut into parts whose (plus, minus)
counters are persisted as they finish and a failed or interrupted run only
recomputes the parts that are missing.

The journal is a JSON-lines file:

* line 1, the header: schema, n, a digest of the matrix, the step range and
  the part count (the parts are the ``split_steps`` edge rule applied to the
  range, so they are a function of the header alone);
* one line per finished part: ``{"part": k, "lo": .., "hi": .., "plus": ..,
  "minus": ..}``, appended and fsync'ed after the part's device work returned.

A journal that does not match the matrix, the range or the part count is
refused (ValueError) rather than silently restarted.  A torn last line (the
process died inside the write) is dropped on load.

Every part runs on the GPU through the same calls as ``perm_chunk`` /
``perm_mod3_parallel`` (several GPUs in one process: ``tp_range_sum_nccl``;
under torch.distributed: ``parallel.distributed_counts``, rank 0 keeps the
journal).  No CPU engine.
"""

from __future__ import annotations

import hashlib
import json
import os
from typing import Callable, Dict, List, Optional, Tuple

from .permanent import MAX_N, SINGLE_LIMB_MAX_N, MatrixF3, _as_matrix, _check_n, _finalize

SCHEMA = "tritperm.ranges.v1"

CountsFn = Callable[[MatrixF3, int, int], Tuple[int, int]]


def matrix_digest(m: MatrixF3) -> str:
    """sha256 of n and the uint8 classes, row-major."""
    h = hashlib.sha256()
    h.update(m.n.to_bytes(2, "little"))
    h.update(m.classes().tobytes())
    return h.hexdigest()


def part_ranges(lo: int, hi: int, parts: int) -> List[Tuple[int, int]]:
    """[lo, hi) cut into `parts` contiguous ranges by the split_steps edge rule
    (src/permanent.py:227-229); empty parts are kept."""
    if parts < 1:
        raise ValueError(f"parts must be >= 1, got {parts}")
    total = hi - lo
    edges = [lo + (total * k) // parts for k in range(parts + 1)]
    return [(edges[k], edges[k + 1]) for k in range(parts)]


class RangeJournal:
    """Append-only record of the finished parts of one traversal."""

    def __init__(self, path: str, m: MatrixF3, lo: int, hi: int, parts: int):
        self.path = path
        self.header = {"schema": SCHEMA, "n": m.n, "matrix_sha256": matrix_digest(m), "lo": lo, "hi": hi,
                       "parts": parts}
        self.ranges = part_ranges(lo, hi, parts)
        self.done: Dict[int, Tuple[int, int]] = {}

    def load(self) -> int:
        """Read an existing journal (if any) and return the number of finished
        parts found.  Raises ValueError when the file belongs to another job."""
        self.done.clear()
        if not os.path.exists(self.path) or os.path.getsize(self.path) == 0:
            return 0
        with open(self.path, encoding="utf-8") as fh:
            lines = fh.read().split("\n")
        torn = lines[-1] != ""  # no trailing newline: the last write did not finish
        body = [ln for ln in (lines[:-1] if torn else lines) if ln.strip()]
        if not body:
            return 0
        try:
            head = json.loads(body[0])
        except json.JSONDecodeError as exc:
            raise ValueError(f"{self.path}: not a {SCHEMA} journal") from exc
        if head != self.header:
            diff = sorted(k for k in set(head) | set(self.header) if head.get(k) != self.header.get(k))
            raise ValueError(f"{self.path}: journal belongs to another job (differs in {', '.join(diff)})")
        for ln in body[1:]:
            try:
                rec = json.loads(ln)
                k, plo, phi, p, q = (int(rec[f]) for f in ("part", "lo", "hi", "plus", "minus"))
            except (json.JSONDecodeError, KeyError, TypeError, ValueError) as exc:
                raise ValueError(f"{self.path}: corrupt record {ln!r}") from exc
            if not 0 <= k < len(self.ranges) or self.ranges[k] != (plo, phi):
                raise ValueError(f"{self.path}: part {k} [{plo}, {phi}) is not a part of this job")
            if p < 0 or q < 0 or p + q > phi - plo:
                raise ValueError(f"{self.path}: part {k} has impossible counters ({p}, {q})")
            if k in self.done and self.done[k] != (p, q):
                raise ValueError(f"{self.path}: part {k} recorded twice with different counters")
            self.done[k] = (p, q)
        if torn:
            self._rewrite()
        return len(self.done)

    def _rewrite(self) -> None:
        tmp = self.path + ".tmp"
        with open(tmp, "w", encoding="utf-8") as fh:
            fh.write(json.dumps(self.header) + "\n")
            for k in sorted(self.done):
                fh.write(self._record(k) + "\n")
            fh.flush()
            os.fsync(fh.fileno())
        os.replace(tmp, self.path)

    def _record(self, k: int) -> str:
        (plo, phi), (p, q) = self.ranges[k], self.done[k]
        return json.dumps({"part": k, "lo": plo, "hi": phi, "plus": p, "minus": q})

    def append(self, k: int, plus: int, minus: int) -> None:
        """Persist part k's counters (header first, on a fresh file)."""
        fresh = not os.path.exists(self.path) or os.path.getsize(self.path) == 0
        self.done[k] = (int(plus), int(minus))
        with open(self.path, "a", encoding="utf-8") as fh:
            if fresh:
                fh.write(json.dumps(self.header) + "\n")
            fh.write(self._record(k) + "\n")
            fh.flush()
            os.fsync(fh.fileno())

    def missing(self) -> List[int]:
        return [k for k in range(len(self.ranges)) if k not in self.done]

    def totals(self) -> Tuple[int, int]:
        return sum(p for p, _ in self.done.values()), sum(q for _, q in self.done.values())


def _default_counts(devices: Optional[List[int]]) -> CountsFn:
    from . import _kernels, parallel

    if parallel.world_size() > 1:
        return lambda m, lo, hi: parallel.distributed_counts(m, lo, hi)

    def counts(m: MatrixF3, lo: int, hi: int) -> Tuple[int, int]:
        mags, sgns = m.planes()
        if devices is not None and len(devices) > 1 and m.n <= SINGLE_LIMB_MAX_N:
            return _kernels.chunk_counts_multi(mags, sgns, m.n, lo, hi, devices)
        return _kernels.chunk_counts(mags, sgns, m.n, lo, hi)

    return counts


def resumable_counts(m, path: str, parts: int = 64, lo: int = 1, hi: Optional[int] = None, jobs=None,
                     max_parts: Optional[int] = None, counts_fn: Optional[CountsFn] = None,
                     on_part: Optional[Callable[[int, int, int], None]] = None) -> Tuple[int, int, bool]:
    """(plus, minus, complete) of steps [lo, hi) with the finished parts kept in
    the journal at `path`.

    Parts already in the journal are not recomputed.  ``max_parts`` bounds the
    parts computed by this call (a time-boxed session); ``complete`` tells
    whether every part is now in the journal.  ``jobs`` is the GPU count of
    ``perm_mod3_parallel``.  ``on_part(k, plus, minus)`` is called after each
    part is persisted.
    """
    from . import parallel

    m = _as_matrix(m)
    _check_n(m.n)
    if hi is None:
        hi = 1 << m.n
    if not 1 <= lo <= hi <= (1 << m.n):
        raise ValueError(f"need 1 <= lo <= hi <= 2**n, got lo={lo} hi={hi} n={m.n}")
    world = parallel.world_size()
    writer = world == 1 or parallel.rank() == 0
    if counts_fn is None:
        devices = None
        if world == 1:
            from .permanent import resolve_gpus

            devices = resolve_gpus(jobs)
        counts_fn = _default_counts(devices)
    journal = RangeJournal(path, m, lo, hi, parts)
    journal.load()
    if world > 1:  # every rank has read the file before rank 0 appends to it
        parallel._dist().barrier()
    computed = 0
    for k in journal.missing():
        if max_parts is not None and computed >= max_parts:
            break
        plo, phi = journal.ranges[k]
        p, q = counts_fn(m, plo, phi) if plo < phi else (0, 0)
        if writer:
            journal.append(k, p, q)
        else:
            journal.done[k] = (int(p), int(q))
        computed += 1
        if on_part is not None:
            on_part(k, int(p), int(q))
    plus, minus = journal.totals()
    return plus, minus, not journal.missing()


def perm_mod3_resumable(m, path: str, parts: int = 64, jobs=None, max_parts: Optional[int] = None,
                        counts_fn: Optional[CountsFn] = None) -> Optional[int]:
    """perm(m) mod 3 (centred) over a journalled full traversal; None while
    parts are still missing (``max_parts`` reached).  Invariant to ``parts``,
    ``jobs`` and to where earlier sessions stopped."""
    m = _as_matrix(m)
    if m.n > MAX_N:
        raise ValueError(f"the B200 engines support n <= {MAX_N}, got n={m.n}")
    plus, minus, complete = resumable_counts(m, path, parts=parts, jobs=jobs, max_parts=max_parts,
                                             counts_fn=counts_fn)
    return _finalize(m.n, plus - minus) if complete else None
