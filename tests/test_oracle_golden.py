"""CPU: the C oracle (oracle/oracle.c) against vectors produced by the
reference itself (tests/golden/*.json, made by tests/golden/make_golden.py).
This pins the checker before any CUDA result is compared with it."""

import random

import numpy as np
import pytest

from conftest import centred, dec, load_golden


def test_chunk_sum_matches_reference_vectors(oracle):
    g = load_golden("chunks.json")
    checked = 0
    for case in g["cases"]:
        n = case["n"]
        mags, sgns = oracle.planes_from_classes(dec(case["a"], n))
        for lo, hi, s in case["ranges"]:
            if hi - lo > (1 << 22) and n > 40:
                continue
            assert oracle.chunk_sum(mags, sgns, n, lo, hi) == s, (n, lo, hi)
            checked += 1
    assert checked > 300


def test_pure_python_restatement_matches_reference(oracle):
    g = load_golden("chunks.json")
    for case in g["cases"]:
        n = case["n"]
        if n > 12:
            continue
        mags, sgns = oracle.planes_from_classes(dec(case["a"], n))
        for lo, hi, s in case["ranges"]:
            assert oracle.py_chunk_sum([int(v) for v in mags], [int(v) for v in sgns], n, lo, hi) == s


def test_oracle_tower(oracle):
    g = load_golden("tower.json")
    for block in g["random"]:
        n = block["n"]
        for s, v, partial in block["mats"][:60]:
            a = dec(s, n)
            assert oracle.perm_centered(a) == v
            assert oracle.partial_full(a) == partial
            if n <= 9:
                assert oracle.perm_ryser(a) == v
            if n <= 6:
                assert oracle.perm_naive(a) == v
    for s, v in g["exhaustive2"]:
        assert oracle.perm_naive(dec(s, 2)) == v


def test_known_values(oracle):
    for s, v in load_golden("anchors.json")["known"]:
        n = int(round(len(s) ** 0.5))
        assert oracle.perm_centered(dec(s, n)) == v


def test_splitmix_golden_words(oracle):
    g = load_golden("rng.json")
    state = 0
    words = []
    for _ in range(3):
        state = (state + oracle.GOLDEN) & oracle.MASK64
        words.append(oracle.py_mix64(state))
    assert words == g["zero_seed_words"]
    assert oracle.lib().orc_mix64(0) == 0


def test_sampler_matches_reference_stream(oracle):
    for case in load_golden("rng.json")["samples"]:
        n = case["n"]
        want = dec(case["entries"], n)
        got = oracle.sample_classes(n, case["seed"], case["trial"])
        assert np.array_equal(got, want), case
        py = np.array(oracle.py_sample_trits(case["seed"], case["trial"], n * n), dtype=np.uint8).reshape(n, n)
        assert np.array_equal(py, want)


def test_mc_zero_count_matches_reference(oracle):
    for case in load_golden("anchors.json")["montecarlo"]:
        assert oracle.mc_zero_count(case["n"], 0, case["trials"], case["seed"]) == case["zero_count"], case


def test_c1_anchors(oracle):
    for case in load_golden("anchors.json")["c1"]:
        a = dec(case["a"], 20)
        assert np.array_equal(a, oracle.sample_classes(20, case["seed"], case["trial"]))
        assert oracle.partial_full(a) == case["partial"]
        assert oracle.perm_centered(a) % 3 == case["class"] == case["ryser_class"]


def test_batch_runner_matches_single(oracle):
    a = np.stack([oracle.sample_classes(9, 3, t) for t in range(40)])
    cls, part = oracle.perm_batch(a, threads=4)
    for b in range(40):
        assert part[b] == oracle.partial_full(a[b])
        assert cls[b] == oracle.perm_centered(a[b]) % 3


def test_threaded_chunk_sum_is_split_invariant(oracle):
    r = random.Random(3)
    for n in (10, 17, 22):
        a = np.array([[r.randrange(3) for _ in range(n)] for _ in range(n)], dtype=np.uint8)
        mags, sgns = oracle.planes_from_classes(a)
        full = oracle.chunk_sum(mags, sgns, n, 1, 1 << n)
        for t in (2, 3, 8):
            assert oracle.chunk_sum_mt(mags, sgns, n, 1, 1 << n, t) == full


@pytest.mark.parametrize("n", [3, 5])
def test_ryser_equals_naive_exhaustive_small(oracle, n):
    r = random.Random(n)
    for _ in range(200):
        a = [[r.randrange(-1, 2) for _ in range(n)] for _ in range(n)]
        assert oracle.perm_ryser(np.mod(a, 3)) == oracle.perm_naive(np.mod(a, 3))


def test_u64_walk_matches_reference_big_int_twin(oracle):
    """n = 63, 64 windows up to 2^64 from the reference's _chunk_sum_pure
    (src/permanent.py:157-178), through the oracle's uint64 restatement."""
    for case in load_golden("n64.json")["cases"]:
        n = case["n"]
        mags, sgns = oracle.planes_from_classes(dec(case["a"], n))
        for lo, hi, s in case["ranges"]:
            p, q = oracle.chunk_counts_u64(mags, sgns, n, lo, hi)
            assert p - q == s, (n, lo, hi)


def test_exhaustive_3x3_naive_vs_ryser(oracle):
    """All 19,683 3x3 matrices: Ryser (oracle) == permutation expansion,
    the reference's exhaustive tower (tests/test_acceptance.py:102-123)."""
    import itertools

    for flat in itertools.product((0, 1, 2), repeat=9):
        a = np.array(flat, dtype=np.int64).reshape(3, 3)
        assert oracle.perm_ryser(a) == oracle.perm_naive(a)
