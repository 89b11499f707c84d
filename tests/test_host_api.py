"""CPU: host-side logic of the product package (no kernel calls): the packed
encoding, the sampler stream, the fixture generators, partition helpers and
argument validation (which, as in the reference, happens before any device
work)."""

import itertools
import os
import re

import numpy as np
import pytest

import paper_2407_20205_b200 as tp
from paper_2407_20205_b200 import _kernels, core_f3, fixtures, rng
from conftest import REPO, dec, load_golden


def test_encode_layout_example():
    g = load_golden("core_ops.json")["encode_example"]
    r = tp.encode(tuple(g["in"]))
    assert (r.mag, r.sgn) == (g["mag"], g["sgn"]) == (0xD, 0x1)


def test_add_sub_match_reference_on_every_pair():
    g = load_golden("core_ops.json")
    for row in g["pairs"]:
        m1, s1, m2, s2 = row["in"]
        a = tp.add_reps(tp.PackedF3Vec(1, m1, s1), tp.PackedF3Vec(1, m2, s2))
        s = tp.sub_reps(tp.PackedF3Vec(1, m1, s1), tp.PackedF3Vec(1, m2, s2))
        assert [a.mag, a.sgn] == row["add"]
        assert [s.mag, s.sgn] == row["sub"]
    for row in g["wide"]:
        m1, s1, m2, s2 = row["in"]
        a = tp.add_reps(tp.PackedF3Vec(32, m1, s1), tp.PackedF3Vec(32, m2, s2))
        assert [a.mag, a.sgn] == row["add"]


def test_walk_add_is_sub_of_negation_on_decoded_values():
    # The kernels add a row as sub of its negation (csrc/tp_device.cuh).
    for v1 in itertools.product((-1, 0, 1), repeat=3):
        for v2 in itertools.product((-1, 0, 1), repeat=3):
            e1, e2 = tp.encode(v1), tp.encode(v2)
            assert tp.decode(tp.sub_reps(e1, core_f3.negate(e2))) == tp.decode(tp.add_reps(e1, e2))


def test_decode_alternate_zero_and_validation():
    assert tp.decode(tp.PackedF3Vec(n=4, mag=0xD, sgn=0x3)) == (1, 1, 0, -1)
    with pytest.raises(ValueError):
        tp.encode(())
    with pytest.raises(ValueError):
        tp.encode((0, 2))
    with pytest.raises(ValueError):
        tp.PackedF3Vec(2, 4, 0)


def test_full_magnitude_and_sign_parity():
    assert tp.is_full_magnitude(tp.encode((1, -1, 1)))
    assert not tp.is_full_magnitude(tp.encode((1, 0, 1)))
    assert tp.sign_parity(tp.encode((-1, -1, 1))) == 1
    assert tp.sign_parity(tp.encode((-1, 1, 1))) == -1


def test_rng_matches_reference_vectors():
    g = load_golden("rng.json")
    state, words = 0, []
    for _ in range(3):
        w, state = rng.next_word(state)
        words.append(w)
    assert words == g["zero_seed_words"]
    for case in g["samples"]:
        n = case["n"]
        want = dec(case["entries"], n)
        got = np.mod(np.array(rng.sample_square(case["seed"], case["trial"], n)), 3)
        assert np.array_equal(got, want)


def test_uniform_fixture_is_the_reference_stream():
    for case in load_golden("rng.json")["samples"]:
        n = case["n"]
        got = fixtures.uniform_batch(n, case["seed"], case["trial"], 1)[0]
        assert np.array_equal(got, dec(case["entries"], n))
    batch = fixtures.uniform_batch(7, 42, 10, 50)
    for k in range(50):
        assert np.array_equal(batch[k], np.mod(np.array(rng.sample_square(42, 10 + k, 7)), 3))


def test_structured_fixture_families():
    e, fam, exp = fixtures.structured_batch(8, 5, 40)
    assert e.shape == (40, 8, 8) and e.dtype == np.uint8
    assert list(np.bincount(fam)) == [10, 10, 10, 10]
    assert (e[fam == 2] == 1).all()
    assert (exp[fam == 2] == 0).all()  # 8! = 40320 = 0 mod 3
    sp = fixtures.sparse_batch(32, 1, 64)
    frac0 = (sp == 0).mean()
    assert 0.77 < frac0 < 0.83
    per, meta = fixtures.perturbed_permutation_batch(9, 3, 30)
    for b in range(30):
        i, j, c, on = meta[b]
        m = per[b].astype(int)
        nz = (m != 0).sum()
        assert nz in (8, 9, 10)
        assert m[i, j] == c


def test_perturbed_permutation_closed_form_small():
    from itertools import permutations

    per, meta = fixtures.perturbed_permutation_batch(5, 11, 40)
    want = fixtures.perturbed_expected(meta)
    for b in range(40):
        a = per[b].astype(int)
        a = np.where(a == 2, -1, a)
        tot = 0
        for s in permutations(range(5)):
            p = 1
            for r, c in enumerate(s):
                p *= a[r, c]
            tot += p
        assert tot % 3 == want[b]


def test_split_steps_and_resolve_jobs():
    for n, jobs in ((1, 4), (5, 1), (5, 31), (5, 100), (20, 7)):
        ranges = tp.split_steps(n, jobs)
        assert len(ranges) == jobs and ranges[0][0] == 1 and ranges[-1][1] == 1 << n
        for (a, b), (c, d) in zip(ranges, ranges[1:]):
            assert a <= b == c <= d
    assert tp.resolve_jobs(5) == 5
    with pytest.raises(ValueError):
        tp.resolve_jobs(0)
    os.environ["TRITPERM_THREADS"] = "3"
    try:
        assert tp.resolve_jobs() == 3
    finally:
        del os.environ["TRITPERM_THREADS"]


def test_matrix_validation_and_normalisation():
    a = tp.MatrixF3([[0, 1], [2, 2]])
    assert a == tp.MatrixF3([[0, 1], [-1, -1]])
    assert a.rows == ((0, 1), (-1, -1))
    assert a.classes().tolist() == [[0, 1], [2, 2]]
    with pytest.raises(ValueError):
        tp.MatrixF3([])
    with pytest.raises(ValueError):
        tp.MatrixF3([[1, 0], [1]])
    mags, sgns = tp.MatrixF3([[1, -1, 0], [0, 0, 1], [-1, 1, 1]]).planes()
    assert mags.tolist() == [0b110, 0b001, 0b111] and sgns.tolist() == [0b010, 0, 0b100]


def test_argument_errors_raise_before_device_work():
    m = tp.MatrixF3([[1, 0, 0, 1]] * 4)
    for lo, hi in ((0, 5), (3, 2), (1, 17)):
        with pytest.raises(ValueError):
            tp.perm_chunk(m, lo, hi)
    with pytest.raises(ValueError):
        tp.montecarlo_zero(0, 10)
    with pytest.raises(ValueError):
        tp.montecarlo_zero(64, 10)
    with pytest.raises(ValueError):
        tp.montecarlo_zero(3, 0)
    with pytest.raises(ValueError):
        tp.perm_mod3_batch(np.zeros((2, 3, 4), dtype=np.uint8))
    with pytest.raises(ValueError):
        tp.perm_mod3_fast(tp.MatrixF3([[1] * 65] * 65))


def test_range_bounds_checked_before_uint64_conversion():
    """2**64 and beyond never reach ctypes (which would wrap them): the bounds
    are Python ints checked first; n = 64 ranges ending at 2**64 are legal
    (tp_range_sum_ex), larger ones and n > 64 are ValueError."""
    z = np.zeros(64, np.uint64)
    for n, lo, hi in ((64, 1, (1 << 64) + 1), (64, 5, 4), (65, 1, 2), (63, 1, 1 << 64), (20, -1, 3)):
        with pytest.raises(ValueError):
            _kernels.chunk_counts(z[:min(n, 64)] if n <= 64 else np.zeros(n, np.uint64),
                                  z[:min(n, 64)] if n <= 64 else np.zeros(n, np.uint64), n, lo, hi)
    with pytest.raises(ValueError):
        _kernels.chunk_counts_multi(z, z, 64, 1, 1 << 64, [0])
    m64 = tp.MatrixF3([[1] * 64] * 64)
    with pytest.raises(ValueError):
        tp.perm_chunk(m64, 0, 1 << 64)
    with pytest.raises(ValueError):
        tp.perm_chunk(m64, 1, (1 << 64) + 1)


def test_rank_split_reaches_two_to_the_64():
    """The rank partition of a 64-row walk (parallel.rank_range) tiles
    [1, 2**64) with the split_steps edge rule in Python ints."""
    from paper_2407_20205_b200 import parallel

    parts = [parallel.rank_range(64, r, 8) for r in range(8)]
    assert parts[0][0] == 1 and parts[-1][1] == 1 << 64
    assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
    assert parts == tp.split_steps(64, 8)


def test_library_exports_every_declared_symbol():
    with open(_kernels.HEADER_PATH) as f:
        header = f.read()
    declared = set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(tp_\w+)\s*\(", header, flags=re.M))
    assert len(declared) >= 14
    assert declared == set(_kernels.SIGNATURES), declared ^ set(_kernels.SIGNATURES)
    L = _kernels.lib()
    for name in declared:
        assert hasattr(L, name), name
    assert L.tp_version() == 200


def test_library_fails_loudly_without_a_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    assert _kernels.device_count() == 0
    with pytest.raises(Exception):
        _kernels.chunk_sum(np.zeros(3, np.uint64), np.zeros(3, np.uint64), 3, 1, 8)
    with pytest.raises(RuntimeError):
        tp.perm_mod3_parallel(tp.MatrixF3([[1, 1], [1, 1]]), jobs=2)


def test_pi_matrix_matches_reference():
    for rec in load_golden("pi.json")["pi_matrix"]:
        n = rec["n"]
        m = tp.pi_matrix(n, skip_integer_part=rec["skip_integer_part"])
        assert np.array_equal(m.classes(), dec(rec["a"], n)), (n, rec["skip_integer_part"])
    assert tp.pi_matrix(3).rows == ((0, 1, 1), (1, -1, 0), (-1, 0, -1))
    with pytest.raises(ValueError):
        tp.pi_matrix(0)
    with pytest.raises(ValueError):
        tp.pi_matrix(101)
    assert tp.pi_matrix(100).n == 100
    with pytest.raises(ValueError):
        tp.pi_matrix(100, skip_integer_part=True)


def test_pi_digits_spot_values():
    from paper_2407_20205_b200 import pi

    d = pi.pi_digits()
    assert len(d) == 10000 and d.startswith("314159265358979323846")
    assert pi.pi_digit(1) == 3 and pi.pi_digit(2) == 1


def test_exact_census_guards():
    with pytest.raises(ValueError):
        tp.exact_zero_count(0)
    with pytest.raises(ValueError):
        tp.exact_zero_count(7)
