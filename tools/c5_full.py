"""The C5 config's own answer: perm mod 3 of the seed-0, trial-0 50x50
matrix (BASELINE.json configs[4]) by the full 2^50-step traversal on one
B200, run twice by two different kernels -- the bucketed walk (default) and
the packed walk (TRITPERM_BUCKET=0) -- plus the 8-part split_steps partition
(src/permanent.py:221-229) that the multi-GPU run uses.  Writes
tests/golden/c5_full.json (the pin of tests/test_gpu_coverage.py) and prints
one JSON record per run.  A CPU oracle would need ~10^6 core-seconds, so the
pin is the agreement of the two kernels; the matrix's 2^36-step window is
oracle-pinned separately (anchors.json c5_window36).

    python tools/c5_full.py [--out tests/golden/c5_full.json] [--skip-packed]
"""
import argparse
import json
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import paper_2407_20205_b200 as tp  # noqa: E402
from paper_2407_20205_b200 import _kernels, fixtures  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--out", default=os.path.join(REPO, "tests", "golden", "c5_full.json"))
ap.add_argument("--skip-packed", action="store_true")
args = ap.parse_args()

a = fixtures.uniform_batch(50, 0, 0, 1)[0]
m = tp.MatrixF3(a.astype("int64"))
mags, sgns = m.planes()
runs = {}
for name, env in (("bucketed", "1"), ("packed", "0")):
    if name == "packed" and args.skip_packed:
        continue
    os.environ["TRITPERM_BUCKET"] = env
    _kernels.walk_tested(0)
    t0 = time.perf_counter()
    p, q = _kernels.chunk_counts(mags, sgns, 50, 1, 1 << 50)
    dt = time.perf_counter() - t0
    rec = {"kernel": name, "plus": p, "minus": q, "partial": p - q, "seconds": round(dt, 2),
           "terms_per_s": (1 << 50) / dt, "tested_pairs": _kernels.walk_tested(0)}
    runs[name] = rec
    print(json.dumps(rec), flush=True)
os.environ["TRITPERM_BUCKET"] = "1"
parts = []
t0 = time.perf_counter()
for lo, hi in tp.split_steps(50, 8):
    parts.append(tp.perm_chunk(m, lo, hi).partial_sum)
dt8 = time.perf_counter() - t0
b = runs["bucketed"]
assert sum(parts) == b["partial"], (parts, b)
if "packed" in runs:
    assert runs["packed"]["plus"] == b["plus"] and runs["packed"]["minus"] == b["minus"], runs
s = b["partial"]
out = {"n": 50, "seed": 0, "trial": 0, "a": "".join(str(int(v)) for v in a.reshape(-1)),
       "plus": b["plus"], "minus": b["minus"], "partial": s, "class": tp.cmod3(s) % 3,
       "parts8": parts, "parts8_seconds": round(dt8, 2),
       "runs": runs, "device": _kernels.device_info(),
       "source": "B200, tools/c5_full.py: bucketed and packed walks agree"}
print(json.dumps({k: v for k, v in out.items() if k != "a"}), flush=True)
os.makedirs(os.path.dirname(args.out), exist_ok=True)
with open(args.out, "w") as f:
    json.dump(out, f, separators=(",", ":"))
    f.write("\n")
