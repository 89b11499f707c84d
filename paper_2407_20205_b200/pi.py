"""Decimal digits of pi and the pi-digit matrices Pi_n (reference:
src/experiments.py:193-213, src/pi_digits.py).

The reference embeds 10,000 digits as data.  Here they are computed with
Machin's formula, pi = 16 atan(1/5) - 4 atan(1/239), in fixed-point integer
arithmetic with guard digits.  tests/golden/pi.json holds the reference's
own pi_matrix(50) rows for both variants, so the two sources are checked
against each other.  Pi_50 is the paper's showcase input: perm(Pi_50) = -1
mod 3, which took 832 h of CPU time there.
"""

from __future__ import annotations

from functools import lru_cache

from .permanent import MatrixF3, cmod3

MAX_DIGITS = 10000  # the reference's embedded table size (src/pi_digits.py:138)


def _atan_inv(x: int, scale: int) -> int:
    """atan(1/x) * scale by the alternating Taylor series."""
    total = term = scale // x
    x2 = x * x
    k = 1
    while term:
        term //= x2
        k += 2
        total += -(term // k) if (k // 2) & 1 else term // k
    return total


@lru_cache(maxsize=4)
def pi_digits(count: int = MAX_DIGITS) -> str:
    """The first `count` digits of pi without the decimal point ("31415...")."""
    guard = 12
    scale = 10 ** (count - 1 + guard)
    pi = (16 * _atan_inv(5, scale) - 4 * _atan_inv(239, scale)) // 10**guard
    # decimal conversion in 1000-digit chunks (int -> str is capped at 4300 digits)
    chunks = []
    base = 10**1000
    while pi:
        pi, r = divmod(pi, base)
        chunks.append(r)
    text = str(chunks[-1]) + "".join(f"{c:01000d}" for c in reversed(chunks[:-1]))
    return text[:count]


def pi_digit(k: int) -> int:
    """The k-th digit (1-based) of pi written without its decimal point."""
    if not 1 <= k <= MAX_DIGITS:
        raise ValueError(f"only {MAX_DIGITS} digits are available, got k={k}")
    return int(pi_digits()[k - 1])


def pi_matrix(n: int, skip_integer_part: bool = False) -> MatrixF3:
    """n-by-n matrix of consecutive digits of pi, row-major, reduced mod 3.

    Starts at the leading "3" unless ``skip_integer_part`` (then at the first
    fractional digit), exactly as src/experiments.py:193-213.
    """
    if n < 1:
        raise ValueError("n must be >= 1")
    offset = 1 if skip_integer_part else 0
    need = n * n + offset
    if need > MAX_DIGITS:
        raise ValueError(f"pi_matrix(n={n}) needs {need} digits but only {MAX_DIGITS} are available")
    d = pi_digits()
    return MatrixF3([[cmod3(int(d[i * n + j + offset])) for j in range(n)] for i in range(n)])
