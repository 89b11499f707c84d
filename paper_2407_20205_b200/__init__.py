"""B200-native Gray-code Ryser permanent mod 3 (arXiv 2407.20205).

Drop-in for the hot path of the reference package ``tritperm``: the same
entry-point names and signatures (``MatrixF3``, ``perm_chunk``,
``perm_mod3_fast``, ``perm_mod3_parallel``, ``split_steps``,
``resolve_jobs``, ``montecarlo_zero``, ``sample_trial_matrix``, ...), with
the traversal in hand-written sm_100a CUDA reached through a C ABI
(include/tritperm.h, lib/libtritperm_b200.so).  No CPU fallback.
"""

from .core_f3 import (
    PackedF3Vec,
    add_reps,
    decode,
    encode,
    is_full_magnitude,
    negate,
    sign_parity,
    sub_reps,
)
from .checkpoint import RangeJournal, perm_mod3_resumable, resumable_counts
from .experiments import (
    ExactCountResult,
    McHistogram,
    McResult,
    exact_zero_count,
    montecarlo_hist,
    montecarlo_zero,
    sample_trial_matrix,
    trial_classes,
)
from .pi import pi_digit, pi_matrix
from .permanent import (
    ChunkResult,
    MatrixF3,
    cmod3,
    perm_chunk,
    perm_mod3_batch,
    perm_mod3_fast,
    perm_mod3_parallel,
    resolve_gpus,
    resolve_jobs,
    split_steps,
)

__version__ = "0.1.0"

__all__ = [
    "ChunkResult",
    "ExactCountResult",
    "MatrixF3",
    "McHistogram",
    "McResult",
    "PackedF3Vec",
    "RangeJournal",
    "add_reps",
    "cmod3",
    "decode",
    "encode",
    "exact_zero_count",
    "is_full_magnitude",
    "montecarlo_hist",
    "montecarlo_zero",
    "negate",
    "perm_chunk",
    "perm_mod3_batch",
    "perm_mod3_fast",
    "perm_mod3_parallel",
    "perm_mod3_resumable",
    "pi_digit",
    "pi_matrix",
    "resolve_gpus",
    "resolve_jobs",
    "resumable_counts",
    "sample_trial_matrix",
    "sign_parity",
    "split_steps",
    "sub_reps",
    "trial_classes",
]
