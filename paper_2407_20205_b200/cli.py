"""Command line, routed to the B200 kernels.

Same subcommands, matrix file format and record schemas as the reference's
``tritperm`` CLI (src/cli.py): ``perm`` (JSON record ``tritperm.perm.v1``),
``count-exact``, ``montecarlo`` (CSV ``tritperm.mc.v1``) and ``pi-matrix``.
Differences: ``perm --method`` accepts only ``mod3`` (the naive and unpacked
engines are CPU oracles, kept with the tests); ``--jobs`` counts GPUs;
``count-exact`` goes to n = 6; ``perm-batch`` is new (one JSON record with
the classes and histogram of a stack of matrices).  Exit status 0, or 1 with
a one-line ``error: ...`` on stderr.

    python -m paper_2407_20205_b200 perm matrix.txt --mod3-classes
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import os
import sys
import time
from typing import List, Optional

PERM_SCHEMA = "tritperm.perm.v1"
MC_SCHEMA = "tritperm.mc.v1"
BATCH_SCHEMA = "tritperm_b200.batch.v1"
MC_COLUMNS = ["schema", "n", "trials", "seed", "zero_count", "p_hat", "stderr"]


def parse_matrix_text(text: str):
    """Matrix file: a size line n, then n lines of n integers (any residues)."""
    from .permanent import MatrixF3

    body = [ln.strip() for ln in text.splitlines() if ln.strip()]
    if not body:
        raise ValueError("matrix file is empty")
    try:
        n = int(body[0])
    except ValueError:
        raise ValueError(f"first line must be the matrix size, got {body[0]!r}") from None
    if n < 1:
        raise ValueError(f"matrix size must be >= 1, got {n}")
    if len(body) != n + 1:
        raise ValueError(f"expected {n} data lines, found {len(body) - 1}")
    rows = []
    for k, line in enumerate(body[1:], start=1):
        fields = line.split()
        if len(fields) != n:
            raise ValueError(f"row {k} has {len(fields)} entries, expected {n}")
        try:
            rows.append([int(f) for f in fields])
        except ValueError:
            raise ValueError(f"row {k} has a non-integer entry: {line!r}") from None
    return MatrixF3(rows)


def format_matrix_text(m, classes: bool = False) -> str:
    lines = [str(m.n)] + [" ".join(str(v % 3 if classes else v) for v in row) for row in m.rows]
    return "\n".join(lines) + "\n"


def _shown(value: int, classes: bool) -> int:
    return value % 3 if classes else value


def _cmd_perm(args) -> int:
    from .permanent import perm_mod3_parallel, resolve_gpus

    if args.method != "mod3":
        raise ValueError(f"method {args.method!r} is a CPU engine; the B200 build provides only 'mod3'")
    with open(args.file, encoding="utf-8") as fh:
        m = parse_matrix_text(fh.read())
    gpus = resolve_gpus(args.jobs)
    t0 = time.perf_counter()
    extra = {}
    if args.checkpoint:
        # journalled traversal: finished parts are kept in the file and a rerun resumes from it
        from .checkpoint import perm_mod3_resumable

        value = perm_mod3_resumable(m, args.checkpoint, parts=args.parts, jobs=len(gpus), max_parts=args.max_parts)
        extra = {"checkpoint": args.checkpoint, "parts": args.parts}
        if value is None:
            print(json.dumps({"schema": PERM_SCHEMA, "n": m.n, "method": "mod3", "jobs": len(gpus), "value": None,
                              "complete": False, "elapsed_seconds": time.perf_counter() - t0, "device": "b200",
                              **extra}))
            return 0
    else:
        value = perm_mod3_parallel(m, len(gpus))
    elapsed = time.perf_counter() - t0
    shown = _shown(value, args.mod3_classes)
    print(shown)
    print(json.dumps({"schema": PERM_SCHEMA, "n": m.n, "method": "mod3", "jobs": len(gpus), "value": shown,
                      "elapsed_seconds": elapsed, "device": "b200", **extra}))
    return 0


def _cmd_perm_batch(args) -> int:
    import numpy as np

    from .permanent import perm_mod3_batch

    arr = np.load(args.file)
    t0 = time.perf_counter()
    cls, _, hist = perm_mod3_batch(arr)
    elapsed = time.perf_counter() - t0
    print(json.dumps({"schema": BATCH_SCHEMA, "batch": int(arr.shape[0]), "n": int(arr.shape[1]),
                      "classes": "".join(str(int(c)) for c in cls), "hist": [int(h) for h in hist],
                      "elapsed_seconds": elapsed}))
    return 0


def _cmd_count_exact(args) -> int:
    from .experiments import exact_zero_count

    r = exact_zero_count(args.n)
    for key, val in (("n", r.n), ("z", r.z), ("total", r.total), ("ratio", f"{r.ratio:.6f}"),
                     ("plus_ones", r.plus_ones), ("minus_ones", r.minus_ones)):
        print(f"{key}: {val}")
    return 0


def _write_csv(columns: List[str], rows: List[dict], out: Optional[str]) -> None:
    if out:
        header = not os.path.exists(out) or os.path.getsize(out) == 0
        with open(out, "a", encoding="utf-8", newline="") as fh:
            w = csv.DictWriter(fh, fieldnames=columns)
            if header:
                w.writeheader()
            w.writerows(rows)
        return
    buf = io.StringIO()
    w = csv.DictWriter(buf, fieldnames=columns)
    w.writeheader()
    w.writerows(rows)
    sys.stdout.write(buf.getvalue())


def _cmd_montecarlo(args) -> int:
    from .experiments import montecarlo_zero

    r = montecarlo_zero(args.n, args.trials, seed=args.seed, jobs=args.jobs)
    _write_csv(MC_COLUMNS, [{"schema": MC_SCHEMA, "n": r.n, "trials": r.trials, "seed": r.seed,
                             "zero_count": r.zero_count, "p_hat": f"{r.p_hat:.9f}",
                             "stderr": f"{r.stderr:.9f}"}], args.out)
    return 0


def _cmd_pi_matrix(args) -> int:
    from .pi import pi_matrix

    text = format_matrix_text(pi_matrix(args.n, skip_integer_part=args.skip_integer_part), args.mod3_classes)
    if args.out:
        with open(args.out, "w", encoding="utf-8") as fh:
            fh.write(text)
    else:
        sys.stdout.write(text)
    return 0


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="tritperm-b200", description="Permanents mod 3 over GF(3) on B200.")
    sub = ap.add_subparsers(dest="command", required=True)

    p = sub.add_parser("perm", help="permanent mod 3 of a matrix file")
    p.add_argument("file")
    p.add_argument("--method", default="mod3")
    p.add_argument("--jobs", type=int, default=None, help="GPUs to split the traversal over")
    p.add_argument("--mod3-classes", action="store_true", help="print {0,1,2} instead of {-1,0,1}")
    p.add_argument("--checkpoint", default=None, help="journal of finished step ranges; a rerun resumes from it")
    p.add_argument("--parts", type=int, default=64, help="parts the traversal is journalled in")
    p.add_argument("--max-parts", type=int, default=None, help="stop after computing this many parts")
    p.set_defaults(func=_cmd_perm)

    p = sub.add_parser("perm-batch", help="classes and histogram of a .npy stack [B, n, n]")
    p.add_argument("file")
    p.set_defaults(func=_cmd_perm_batch)

    p = sub.add_parser("count-exact", help="exact census of perm mod 3 over all n x n matrices (n <= 6)")
    p.add_argument("--n", type=int, required=True)
    p.set_defaults(func=_cmd_count_exact)

    p = sub.add_parser("montecarlo", help="zero-permanent frequency over random matrices")
    p.add_argument("--n", type=int, required=True)
    p.add_argument("--trials", type=int, default=100000)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--jobs", type=int, default=None)
    p.add_argument("--out", default=None, help="append the CSV row to this file")
    p.set_defaults(func=_cmd_montecarlo)

    p = sub.add_parser("pi-matrix", help="write the n x n pi-digit matrix")
    p.add_argument("--n", type=int, required=True)
    p.add_argument("--out", default=None)
    p.add_argument("--skip-integer-part", action="store_true")
    p.add_argument("--mod3-classes", action="store_true")
    p.set_defaults(func=_cmd_pi_matrix)
    return ap


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return args.func(args)
    except (ValueError, OSError, RuntimeError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
