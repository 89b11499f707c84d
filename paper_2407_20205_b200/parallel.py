"""Multi-GPU split of one traversal: one process per GPU, one NCCL all-reduce.

Replaces the reference's ThreadPool fan-out + Python ``sum`` over
``split_steps`` ranges (src/permanent.py:232-255, and
src/experiments.py:182-189 for trials).  Rank r of W takes part r of
``split_steps(n, W)``, accumulates its (plus, minus) counters on its own
device, and the ranks meet in a single ``all_reduce(SUM)`` of a 2-element
int64 tensor -- the only collective on the path (payload 16 bytes, latency
bound; NVLink bandwidth is irrelevant).  Batches shard matrices across ranks
and all-reduce the 3-bin histogram the same way.

The per-rank compute is injectable so the partitioning and the collective
can be tested on CPU with the gloo backend (tests/test_parallel_gloo.py).
"""

from __future__ import annotations

from typing import Callable, Optional, Sequence, Tuple

import numpy as np

CountsFn = Callable[[object, int, int], Tuple[int, int]]


def _dist():
    import torch.distributed as dist

    return dist


def world_size() -> int:
    try:
        dist = _dist()
    except Exception:  # pragma: no cover - torch always present in this image
        return 1
    if dist.is_available() and dist.is_initialized():
        return dist.get_world_size()
    return 1


def rank() -> int:
    dist = _dist()
    return dist.get_rank() if dist.is_available() and dist.is_initialized() else 0


def rank_range(n: int, r: int, w: int, lo: int = 1, hi: Optional[int] = None) -> Tuple[int, int]:
    """Part r of W of steps [lo, hi) with the split_steps edge rule."""
    if hi is None:
        hi = 1 << n
    total = hi - lo
    return lo + (total * r) // w, lo + (total * (r + 1)) // w


def _device_counts(m, lo: int, hi: int) -> Tuple[int, int]:
    from . import _kernels

    mags, sgns = m.planes()
    return _kernels.chunk_counts(mags, sgns, m.n, lo, hi)


def _allreduce_int64(values: Sequence[int], device) -> np.ndarray:
    import torch

    dist = _dist()
    t = torch.tensor([int(v) for v in values], dtype=torch.int64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return t.cpu().numpy()


def distributed_counts(m, lo: int = 1, hi: Optional[int] = None, counts_fn: Optional[CountsFn] = None,
                       device=None) -> Tuple[int, int]:
    """(plus, minus) of steps [lo, hi) summed over all ranks (one all-reduce).

    The counters are exact and below 2^63 for n <= 62, so int64 SUM is exact.
    """
    import torch

    if hi is None:
        hi = 1 << m.n
    w, r = world_size(), rank()
    plo, phi = rank_range(m.n, r, w, lo, hi)
    fn = counts_fn or _device_counts
    p, q = fn(m, plo, phi) if plo < phi else (0, 0)
    if device is None:
        dist = _dist()
        device = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" else "cpu"
    out = _allreduce_int64([p, q], device)
    return int(out[0]), int(out[1])


def perm_mod3_distributed(m, counts_fn: Optional[CountsFn] = None, device=None) -> int:
    """perm(m) mod 3 (centred) with the step range split across ranks."""
    from .permanent import _as_matrix, _finalize

    m = _as_matrix(m)
    p, q = distributed_counts(m, 1, 1 << m.n, counts_fn=counts_fn, device=device)
    return _finalize(m.n, p - q)


def shard_rows(B: int, r: int, w: int) -> Tuple[int, int]:
    """Matrices [b0, b1) of a B-batch owned by rank r (the _split_trials rule,
    src/experiments.py:143-145)."""
    return (B * r) // w, (B * (r + 1)) // w


def distributed_hist(local_hist: Sequence[int], device=None) -> np.ndarray:
    """All-reduce of a rank's 3-bin class histogram."""
    import torch

    if device is None:
        dist = _dist()
        device = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" else "cpu"
    return _allreduce_int64(local_hist, device)
