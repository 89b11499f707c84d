"""GPU parity, second block: the full C3 config, the bucketed walk at n = 30 and
n = 32 (partial pieces, padding-free slots, dummy-slot masks), the exhaustive
3x3 tower, n = 64 windows, Monte Carlo and batches beyond the old list-
workspace cap, concurrent async calls on two streams, the NCCL all-reduce
behind the C ABI, and the full 2^50 traversal of the C5 config matrix."""

import itertools
import os
import random

import numpy as np
import pytest

from conftest import GOLDEN, centred, dec, load_golden

pytestmark = pytest.mark.gpu


def _has(name):
    return os.path.exists(os.path.join(GOLDEN, name))


def test_c3_all_4096_classes_and_histogram(gpu):
    """Config C3 in full: every class and the histogram against
    tests/golden/c3.json (uniform + sparse families from the C oracle, 12
    matrices cross-pinned by the reference's perm_mod3_parallel; all-ones and
    perturbed permutations from their closed forms), and the raw partials of
    all 2,048 oracle matrices.  All of it runs through the bucketed walk
    (17-row A side, 3 key columns, n = 32: no padding column)."""
    if not _has("c3.json"):
        pytest.skip("C3 goldens not generated")
    from paper_2407_20205_b200 import _kernels, fixtures

    g = load_golden("c3.json")
    entries, fam, exp = fixtures.structured_batch(32, 0, 4096)
    import hashlib

    assert hashlib.sha256(entries.tobytes()).hexdigest() == g["entries_sha256"]
    _kernels.walk_tested(0)
    cls, part, hist = gpu.perm_mod3_batch(entries)
    assert _kernels.walk_tested(0) > 0, "bucketed walk not used"
    want = np.frombuffer(g["classes"].encode(), dtype=np.uint8) - ord("0")
    assert np.array_equal(cls, want)
    assert hist.tolist() == g["hist"]
    for i, p in g["partials_oracle"].items():
        assert part[int(i)] == p, i
    known = exp >= 0
    assert np.array_equal(cls[known], exp[known])


def _oracle_partials(oracle, e):
    _, part = oracle.perm_batch(e, threads=os.cpu_count() or 4)
    return part


def test_bucketed_walk_n30_n32_against_oracle(gpu, oracle):
    """n = 32 is the one width where the bucketed walk has no padding column
    (dummy slots are the zero vector, masked by vmask, and the exact fold
    takes the h.x == 0 correction); n = 30 keeps the padding column.  Uniform,
    sparse (partly filled pieces), all-ones (dense mode) and a filter-heavy
    matrix, raw partials against the C oracle."""
    from math import comb

    from paper_2407_20205_b200 import _kernels

    r = np.random.default_rng(3032)
    for n in (30, 32):
        uni = r.integers(0, 3, (3, n, n)).astype(np.uint8)
        sp = ((r.random((2, n, n)) < 0.3) * r.integers(1, 3, (2, n, n))).astype(np.uint8)
        heavy = r.integers(0, 3, (1, n, n)).astype(np.uint8)
        heavy[:, :, n - 16:] = 1  # the 16-column filter passes 2/3 of the pairs
        e = np.concatenate([uni, sp, heavy, np.ones((1, n, n), np.uint8)])
        _kernels.walk_tested(0)
        cls, part, hist = gpu.perm_mod3_batch(e)
        assert _kernels.walk_tested(0) > 0, n
        want = _oracle_partials(oracle, e[:-1])
        assert np.array_equal(part[:-1], want), n
        ones = sum(comb(n, k) * (-1) ** k * (1 if k % 3 == 1 else (-1) ** n) for k in range(n + 1) if k % 3)
        assert part[-1] == ones and cls[-1] == 0, n
        assert hist.sum() == len(e)


def test_exhaustive_3x3_tower(gpu, oracle):
    """All 19,683 3x3 matrices through perm_mod3_batch (the reference's
    exhaustive tower, tests/test_acceptance.py:102-123) against permutation
    expansion."""
    flat = np.array(list(itertools.product((0, 1, 2), repeat=9)), dtype=np.uint8)
    e = flat.reshape(-1, 3, 3)
    cls, part, hist = gpu.perm_mod3_batch(e)
    want = np.array([oracle.perm_naive(a) % 3 for a in e.astype(np.int64)], dtype=np.int8)
    assert np.array_equal(cls, want)
    assert hist.tolist() == np.bincount(want, minlength=3).tolist()
    # and one matrix at a time through the range path, a sample
    for i in range(0, len(e), 997):
        assert gpu.perm_mod3_fast(gpu.MatrixF3(centred(e[i]))) % 3 == want[i]


def test_n64_windows_against_reference_twin(gpu, oracle):
    """perm_chunk at n = 63 and 64: windows up to the end 2^64 pinned by the
    reference's big-int twin (tests/golden/n64.json), and 2^27-step windows
    (the bucketed walk's aligned middle plus generic head and tail, one of
    them ending at 2^64) against the oracle's uint64 walk."""
    from paper_2407_20205_b200 import _kernels

    for case in load_golden("n64.json")["cases"]:
        n = case["n"]
        m = gpu.MatrixF3(centred(dec(case["a"], n)))
        for lo, hi, s in case["ranges"]:
            assert gpu.perm_chunk(m, lo, hi).partial_sum == s, (n, lo, hi)
    r = random.Random(64)
    for case in load_golden("n64.json")["cases"][3:]:
        n = case["n"]
        a = dec(case["a"], n)
        mags, sgns = oracle.planes_from_classes(a)
        m = gpu.MatrixF3(centred(a))
        last = 1 << n
        for lo, hi in ((last - (1 << 27) - 12345, last), (r.randrange(1, last >> 1), None)):
            hi = hi or lo + (1 << 27) + 777
            p, q = oracle.chunk_counts_u64(mags, sgns, n, lo, hi)
            _kernels.walk_tested(0)
            assert gpu.perm_chunk(m, lo, hi).partial_sum == p - q, (n, lo, hi)
            assert _kernels.walk_tested(0) > 0


def test_large_batches_take_the_bucketed_walk(gpu, oracle):
    """No workspace cap: Monte Carlo at n = 28 with 100,000 trials and a
    16,384 x 32 batch both run the bucketed walk (round 1 fell back to the
    packed walk above 6,758 matrices at n >= 28).  The batch's first 1,024
    matrices are C3's uniform family: their classes equal the C3 goldens."""
    from paper_2407_20205_b200 import _kernels, fixtures

    _kernels.walk_tested(0)
    h = gpu.montecarlo_hist(28, 100_000, 11)
    assert _kernels.walk_tested(0) > 0
    assert h.zeros + h.plus_ones + h.minus_ones == 100_000
    # the tally is split-invariant: two halves with their own trial offsets
    c0 = _kernels.mc_hist(28, 0, 50_000, 11)
    c1 = _kernels.mc_hist(28, 50_000, 100_000, 11)
    assert (c0 + c1).tolist() == [h.zeros, h.plus_ones, h.minus_ones]
    e = fixtures.uniform_batch(32, 0, 0, 16384)
    _kernels.walk_tested(0)
    cls, part, hist = gpu.perm_mod3_batch(e)
    assert _kernels.walk_tested(0) > 0
    assert hist.sum() == 16384
    if _has("c3.json"):
        want = np.frombuffer(load_golden("c3.json")["classes"].encode(), dtype=np.uint8) - ord("0")
        assert np.array_equal(cls[:1024], want[:1024])
    want = _oracle_partials(oracle, e[1024:1028])
    assert np.array_equal(part[1024:1028], want)


def test_async_calls_on_two_streams_do_not_share_memory(gpu, oracle):
    """Two tp_walk_async calls with different batches enqueued back to back on
    two streams (no synchronisation between them), twice, then a third on the
    first stream: every count equals the synchronous path's.  Round 1 shared
    one bucket-list workspace per device between them."""
    import torch

    from paper_2407_20205_b200 import _kernels, fixtures

    jobs = [(fixtures.uniform_batch(24, 21, 0, 600), 24), (fixtures.uniform_batch(28, 22, 0, 40), 28),
            (fixtures.uniform_batch(26, 23, 0, 90), 26)]
    want = []
    for e, n in jobs:
        _, part, _ = gpu.perm_mod3_batch(e)
        want.append(part)
    streams = [torch.cuda.Stream(), torch.cuda.Stream(), None]
    streams[2] = streams[0]
    bufs = []
    for e, n in jobs:
        B = len(e)
        d_e = torch.from_numpy(e).cuda()
        d_rows = torch.empty((B, _kernels.ROWREC_BYTES), dtype=torch.uint8, device="cuda")
        d_pm = torch.zeros((B, 2), dtype=torch.int64, device="cuda")
        _kernels.pack_async(d_e.data_ptr(), B, n, d_rows.data_ptr(), torch.cuda.current_stream().cuda_stream)
        bufs.append((d_e, d_rows, d_pm))
    torch.cuda.synchronize()
    for _ in range(2):
        for (e, n), (_, d_rows, d_pm), st in zip(jobs, bufs, streams):
            d_pm.zero_()
        torch.cuda.synchronize()
        for (e, n), (_, d_rows, d_pm), st in zip(jobs, bufs, streams):
            _kernels.walk_async(d_rows.data_ptr(), len(e), n, d_pm.data_ptr(), st.cuda_stream)
        torch.cuda.synchronize()
        for (_, _, d_pm), w in zip(bufs, want):
            pm = d_pm.cpu().numpy()
            assert np.array_equal(pm[:, 0] - pm[:, 1], w)


def test_nccl_all_reduce_behind_the_abi(gpu, oracle):
    """tp_range_sum_nccl: the split of one range across the listed devices
    with the counters summed by ONE ncclAllReduce inside the library (a
    1-device clique on a 1-GPU box; every visible device otherwise), equal to
    tp_range_sum and the host-summing tp_range_sum_multi."""
    from paper_2407_20205_b200 import _kernels

    devs = list(range(max(1, _kernels.device_count())))
    g = load_golden("anchors.json")
    for key in ("c4_window", "c5_window"):
        w = g[key]
        m = gpu.MatrixF3(centred(dec(w["a"], w["n"])))
        mags, sgns = m.planes()
        p, q = _kernels.chunk_counts_multi(mags, sgns, w["n"], w["lo"], w["hi"], devs, nccl=True)
        assert p - q == w["partial"]
        assert (p, q) == _kernels.chunk_counts_multi(mags, sgns, w["n"], w["lo"], w["hi"], devs, nccl=False)
        assert (p, q) == _kernels.chunk_counts(mags, sgns, w["n"], w["lo"], w["hi"])
    case = g["c1"][0]
    m = gpu.MatrixF3(centred(dec(case["a"], 20)))
    assert gpu.perm_mod3_parallel(m, jobs=8) % 3 == case["class"]


def test_c5_config_full_traversal(gpu):
    """The C5 config's own answer: the full 2^50-step traversal of the seed-0,
    trial-0 50x50 matrix (~50 s), and the same range in 8 split_steps parts
    (the multi-GPU partition rule), against tests/golden/c5_full.json.  That
    value was measured on B200 by two different kernels (the bucketed walk
    and the packed walk, TRITPERM_BUCKET=0; tools/c5_full.py) -- a CPU oracle
    would need ~10^6 core-seconds -- and its 2^36-step windows are oracle-
    pinned (anchors.json c5_window36)."""
    if not _has("c5_full.json"):
        pytest.skip("c5_full.json not recorded yet (tools/c5_full.py)")
    g = load_golden("c5_full.json")
    m = gpu.MatrixF3(centred(dec(g["a"], 50)))
    assert gpu.perm_chunk(m, 1, 1 << 50).partial_sum == g["partial"]
    parts = [gpu.perm_chunk(m, lo, hi).partial_sum for lo, hi in gpu.split_steps(50, 8)]
    assert sum(parts) == g["partial"]
    assert parts == g["parts8"]
    assert gpu.perm_mod3_fast(m) % 3 == g["class"]


def test_bounds_checked_build_runs_every_walk_family():
    """Stand-in for compute-sanitizer (closed on this GPU pool: runs under it
    left GPUs needing a reset): the TP_CHECKED build of the library traps on
    any out-of-range table, list or shared-memory index of the bucketed walk
    (RunCursor decode, piece table, pass-list steps, grouping ranks), and
    tools/sanitize_case.py drives every walk family through it against the
    oracle in a separate process."""
    import subprocess
    import sys

    from conftest import REPO

    lib = os.path.join(REPO, "paper_2407_20205_b200", "lib", "checked", "libtritperm_b200.so")
    if not os.path.exists(lib):
        pytest.skip("checked build missing (make -C paper_2407_20205_b200/csrc checked)")
    env = dict(os.environ, TRITPERM_LIB=lib)
    out = subprocess.run([sys.executable, os.path.join(REPO, "tools", "sanitize_case.py")], env=env,
                         capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]
    assert "sanitize case ok" in out.stdout


def test_walk_options_agree(gpu, oracle, monkeypatch):
    """The scheduling and kernel options give the same raw partials: sticky
    pieces off / by the rule / always (n > 32), and the round-2 k_walk_bucket
    (TRITPERM_BATCH=0) against k_walk_batch, on the C4 config's full 2^36
    traversal, the C5 matrix's 2^36-step window, and the C2 batch's first 64
    matrices (all pinned to the reference: anchors.json)."""
    from paper_2407_20205_b200 import _kernels, fixtures

    g = load_golden("anchors.json")
    w4, w5 = g["c4_full"], g["c5_window36"]
    m4 = gpu.MatrixF3(centred(dec(w4["a"], 36)))
    m5 = gpu.MatrixF3(centred(dec(w5["a"], 50)))
    c2 = fixtures.uniform_batch(24, 0, 0, 64)
    for env in ({"TRITPERM_STICKY": "0"}, {"TRITPERM_STICKY": "1"}, {"TRITPERM_STICKY": "2"},
                {"TRITPERM_BATCH": "0"}):
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        _kernels.walk_tested(0)
        assert gpu.perm_chunk(m4, 1, 1 << 36).partial_sum == w4["partial"], env
        assert gpu.perm_chunk(m5, w5["lo"], w5["hi"]).partial_sum == w5["partial"], env
        _, part, _ = gpu.perm_mod3_batch(c2)
        assert part.tolist() == g["c2_partials_head"], env
        assert _kernels.walk_tested(0) > 0, env  # the bucketed walks ran
        for k in env:
            monkeypatch.delenv(k)


def test_filter_list_lengths_and_dense_passes(gpu, oracle):
    """The batched walk's filter takes its list six, three, two or one entries
    at a time, and its pass records are compacted and verified across the
    lanes.  Inputs that push both to their edges, raw partials against the C
    oracle: B-side rows with no entry on the key columns (every state of a
    superblock has the same key trits: lists of 0 or all 128 steps), with
    few entries there (ragged list lengths), filter-heavy rows (the low 16
    columns all ones: the pass lists fill and overflow into the exact path)
    and sparse rows (short pieces, many passes per record); and the group
    kernel's forced rows: columns with a single nonzero entry (subsets
    without that row stay out of the tables), zero columns (empty tables),
    permutation-like matrices.  n = 24 (14-row A side, six-entry loop), n = 29
    (17 rows, three-entry loop) in full, and n = 36 windows (wide kernel)."""
    from paper_2407_20205_b200 import _kernels

    r = np.random.default_rng(2407)

    def family(n, fix, count):
        out = []
        for v in range(count):
            a = r.integers(0, 3, (n, n)).astype(np.uint8)
            keys = slice(0, 5)  # the key columns are the leading columns of the (primary) word
            if v % 8 == 4:  # forced rows: columns with a single nonzero entry (A side, B side), or none
                for c, row in ((7, 2), (9, fix + 1), (12, n - 1)):
                    a[:, c] = 0
                    a[row, c] = 1 + (v // 8 + c) % 2
                if v % 16 == 12:
                    a[:, 11] = 0
            elif v % 8 == 5:  # a permutation matrix with a few extra entries
                a[:] = 0
                a[np.arange(n), r.permutation(n)] = r.integers(1, 3, n)
                a[r.integers(0, n, 3), r.integers(0, n, 3)] = 1
            elif v % 4 == 0:
                a[fix:, keys] = 0
            elif v % 4 == 1:
                a[fix:, keys] = 0
                a[fix + (v // 4) % (n - fix), 0] = 1 + v % 2
            elif v % 4 == 2:
                a[:, n - 16:] = 1
                a[fix:, keys] = (r.random((n - fix, 5)) < 0.3) * r.integers(1, 3, (n - fix, 5))
            else:
                a = ((r.random((n, n)) < 0.25) * r.integers(1, 3, (n, n))).astype(np.uint8)
            out.append(a)
        return np.stack(out)

    for n, fix, count in ((24, 14, 16), (29, 17, 6)):
        e = family(n, fix, count)
        _kernels.walk_tested(0)
        _, part, _ = gpu.perm_mod3_batch(e)
        assert _kernels.walk_tested(0) > 0, n
        assert np.array_equal(part, _oracle_partials(oracle, e)), n
    # n = 36: 2^28-step windows of each matrix (the bucketed walk takes the aligned middle)
    n = 36
    e = family(n, 17, 14)
    for k, a in enumerate(e):
        m = gpu.MatrixF3(centred(a))
        mags, sgns = oracle.planes_from_classes(a)
        lo = (1 << 33) + (k << 29) + 1000 * k
        hi = lo + (1 << 28) + 77
        _kernels.walk_tested(0)
        got = gpu.perm_chunk(m, lo, hi).partial_sum
        # (a zero column or forced rows can leave the tables without a pair to test)
        assert _kernels.walk_tested(0) > 0 or k % 8 in (4, 5), k
        assert got == oracle.chunk_sum_mt(mags, sgns, n, lo, hi, 8), k


def test_table4_tool_small_scale(gpu):
    """tools/table4.py (the paper's Monte Carlo table through montecarlo_zero)
    at 10^-6 of the paper's trial counts: every n = 6..30 runs, the records
    carry the paper's tallies, and the n = 6 frequency sits at the calibration
    value 0.3546 (tests/test_acceptance.py:143-158)."""
    import json
    import subprocess
    import sys

    from conftest import REPO

    out = subprocess.run([sys.executable, os.path.join(REPO, "tools", "table4.py"), "--scale", "1e-6"],
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    recs = [json.loads(ln) for ln in out.stdout.splitlines() if ln.startswith("{")]
    rows = {r["n"]: r for r in recs if "n" in r}
    assert sorted(rows) == list(range(6, 31))
    assert rows[6]["trials"] == 100000 and abs(rows[6]["zero_fraction"] - 0.35456) < 0.01
    assert rows[24]["paper_zero_count"] == 3333518 and rows[30]["trials"] == 1
    # the same call through the API gives the same tally (seed 0)
    assert rows[10]["zero_count"] == gpu.montecarlo_zero(10, rows[10]["trials"], seed=0).zero_count
    assert "summary" in recs[-1]


def test_wide_batch_above_4096_matrices_uses_four_keys(gpu, oracle):
    """n > 32 batches of more than 4,096 matrices take the 4-key tables (26.6 KB
    of run starts per matrix instead of 237 KB) and so another instantiation
    of the batched walk than single matrices and small batches (5 keys).  A
    batch of 4,100 33x33 matrices (mostly sparse, so the traversals are
    short on events but every piece and batch is walked): the first 48 raw
    partials against the same matrices as a small batch (the 5-key kernel),
    three of them against the C oracle's full 2^33 traversal."""
    from paper_2407_20205_b200 import _kernels

    n, B = 33, 4100
    r = np.random.default_rng(3317)
    e = ((r.random((B, n, n)) < 0.3) * r.integers(1, 3, (B, n, n))).astype(np.uint8)
    e[:16] = r.integers(0, 3, (16, n, n))  # uniform
    e[16] = 1                              # all-ones: weighted
    e[17, :, 20:] = 1                      # filter-heavy
    _kernels.walk_tested(0)
    _, part, hist = gpu.perm_mod3_batch(e)
    assert _kernels.walk_tested(0) > 0
    assert hist.sum() == B
    _, small, _ = gpu.perm_mod3_batch(e[:48])
    assert np.array_equal(part[:48], small)
    for k in (0, 17, 40):
        mags, sgns = oracle.planes_from_classes(e[k])
        assert part[k] == oracle.chunk_sum_mt(mags, sgns, n, 1, 1 << n, os.cpu_count() or 8), k
