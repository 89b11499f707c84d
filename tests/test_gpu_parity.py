"""GPU parity: the sm_100a path (through the C ABI) against the reference's
golden vectors and the pinned C oracle, bit-exact on raw partial sums,
classes and histograms."""

import random

import numpy as np
import pytest

from conftest import centred, dec, load_golden

pytestmark = pytest.mark.gpu


def _rand_matrix(r, n):
    return np.array([[r.randrange(3) for _ in range(n)] for _ in range(n)], dtype=np.uint8)


def test_device_primitives_match_reference_tables(gpu):
    from paper_2407_20205_b200 import _kernels

    g = load_golden("core_ops.json")
    rows = g["pairs"] + g["wide"]
    words = np.array([r["in"] for r in rows], dtype=np.uint32)
    add = _kernels.selftest_ops(words, 0)
    sub = _kernels.selftest_ops(words, 1)
    walk_add = _kernels.selftest_ops(words, 2)
    for k, r in enumerate(rows):
        assert add[k].tolist() == r["add"], r  # bit-exact incl. zero-sign bits
        assert sub[k].tolist() == r["sub"], r
        # walk ADD (sub of the negated row): same trits, sign bits free on zeros
        mag = int(walk_add[k, 0])
        assert mag == r["add"][0]
        assert (int(walk_add[k, 1]) & mag) == (r["add"][1] & mag)


def test_chunk_sum_golden_ranges(gpu):
    from paper_2407_20205_b200 import _kernels

    for case in load_golden("chunks.json")["cases"]:
        n = case["n"]
        m = gpu.MatrixF3(centred(dec(case["a"], n)))
        mags, sgns = m.planes()
        for lo, hi, s in case["ranges"]:
            assert _kernels.chunk_sum(mags, sgns, n, lo, hi) == s, (n, lo, hi)
            if lo >= 1:
                assert gpu.perm_chunk(m, lo, hi).partial_sum == s


def test_random_ranges_against_oracle(gpu, oracle):
    r = random.Random(99)
    for n in list(range(1, 40)) + [44, 50, 57, 62, 63]:
        a = _rand_matrix(r, n)
        mags, sgns = oracle.planes_from_classes(a)
        m = gpu.MatrixF3(centred(a))
        last = 1 << n
        for _ in range(5):
            span = min(last, 1 << r.choice((5, 9, 14, 19)))
            lo = r.randrange(0, last - span + 1)
            hi = lo + r.randrange(0, span + 1)
            lo = max(lo, 1)
            hi = max(hi, lo)
            want = oracle.chunk_sum(mags, sgns, n, lo, hi)
            assert gpu.perm_chunk(m, lo, hi).partial_sum == want, (n, lo, hi)


def test_superblock_aligned_windows(gpu, oracle):
    """Windows that exercise the fast kernel's chunking, replay and entry steps."""
    r = random.Random(5)
    for n in (12, 13, 16, 20, 25, 32, 33, 34, 40, 48, 62):
        a = _rand_matrix(r, n)
        mags, sgns = oracle.planes_from_classes(a)
        m = gpu.MatrixF3(centred(a))
        for shift in (12, 13, 17):
            if shift > n:
                continue
            span = 1 << min(shift + 3, n - 1, 21)
            base = (r.randrange(0, (1 << n) - span + 1) >> shift) << shift
            for lo, hi in ((base, base + span), (base + 1, base + span - 1), (base + 31, base + span + 33)):
                lo, hi = max(lo, 1), min(hi, 1 << n)
                if lo > hi:
                    continue
                assert gpu.perm_chunk(m, lo, hi).partial_sum == oracle.chunk_sum(mags, sgns, n, lo, hi), (n, lo, hi)


def test_empty_and_edge_ranges(gpu):
    m = gpu.MatrixF3([[1, -1, 0], [1, 1, 1], [0, 1, -1]])
    assert gpu.perm_chunk(m, 5, 5).partial_sum == 0
    assert gpu.perm_chunk(m, 8, 8).partial_sum == 0
    full = gpu.perm_chunk(m, 1, 8).partial_sum
    assert sum(gpu.perm_chunk(m, lo, hi).partial_sum for lo, hi in gpu.split_steps(3, 5)) == full


def test_oracle_tower_on_gpu(gpu):
    g = load_golden("tower.json")
    for block in g["random"]:
        n = block["n"]
        mats = block["mats"]
        batch = np.stack([dec(s, n) for s, _, _ in mats])
        cls, part, hist = gpu.perm_mod3_batch(batch)
        want = np.array([v % 3 for _, v, _ in mats])
        assert np.array_equal(cls, want)
        assert np.array_equal(part, np.array([p for _, _, p in mats]))
        assert hist.tolist() == np.bincount(want, minlength=3).tolist()
        for s, v, _ in mats[:25]:
            m = gpu.MatrixF3(centred(dec(s, n)))
            assert gpu.perm_mod3_fast(m) == v
            for jobs in (1, 2, 4, 7):
                assert gpu.perm_mod3_parallel(m, jobs=jobs) == v
    for s, v in g["exhaustive2"]:
        assert gpu.perm_mod3_fast(gpu.MatrixF3(centred(dec(s, 2)))) == v


def test_known_values(gpu):
    assert gpu.perm_mod3_fast(gpu.MatrixF3([[1, 0, 0], [0, 1, 0], [0, 0, 1]])) == 1
    assert gpu.perm_mod3_fast(gpu.MatrixF3([[1, 1], [1, 1]])) == -1
    assert gpu.perm_mod3_fast(gpu.MatrixF3([[0]])) == 0
    assert gpu.perm_mod3_fast(gpu.MatrixF3([[-1]])) == -1


def test_device_sampler_matches_reference_stream(gpu):
    from paper_2407_20205_b200 import _kernels, fixtures

    for case in load_golden("rng.json")["samples"]:
        n = case["n"]
        want = dec(case["entries"], n)
        got = _kernels.mc_sample_entries(n, case["trial"], case["seed"]).reshape(n, n)
        assert np.array_equal(np.mod(got.astype(int), 3), want)
    batch = _kernels.sample_classes(24, 0, 300, 7)
    assert np.array_equal(batch, fixtures.uniform_batch(24, 7, 0, 300))


def test_montecarlo_matches_reference_tallies(gpu):
    for case in load_golden("anchors.json")["montecarlo"]:
        r = gpu.montecarlo_zero(case["n"], case["trials"], seed=case["seed"])
        assert r.zero_count == case["zero_count"], case
        assert r.n == case["n"] and r.trials == case["trials"]


def test_montecarlo_hist_matches_oracle_classes(gpu, oracle):
    for n, trials, seed in ((3, 500, 2), (7, 300, 8), (13, 200, 1), (16, 400, 3), (18, 200, 5), (21, 64, 4)):
        h = gpu.montecarlo_hist(n, trials, seed)
        cls, _ = oracle.perm_batch(oracle.sample_batch(n, seed, 0, trials), threads=8)
        assert [h.zeros, h.plus_ones, h.minus_ones] == np.bincount(cls, minlength=3).tolist()
        per = gpu.trial_classes(n, 0, trials, seed)
        assert np.array_equal(per, cls)


def test_c1_anchors(gpu):
    for case in load_golden("anchors.json")["c1"]:
        a = dec(case["a"], 20)
        m = gpu.MatrixF3(centred(a))
        assert gpu.perm_chunk(m, 1, 1 << 20).partial_sum == case["partial"]
        assert gpu.perm_mod3_fast(m) % 3 == case["class"] == case["ryser_class"]
        cls, part, _ = gpu.perm_mod3_batch(a[None])
        assert cls[0] == case["class"] and part[0] == case["partial"]


def test_c2_batch_full(gpu):
    """16,384 x 24x24: every class and the histogram, vs the oracle goldens
    (pinned by the reference's own montecarlo_zero tally)."""
    g = load_golden("anchors.json")
    if "c2_classes" not in g:
        pytest.skip("slow goldens not generated")
    from paper_2407_20205_b200 import fixtures

    entries = fixtures.uniform_batch(24, 0, 0, 16384)
    cls, part, hist = gpu.perm_mod3_batch(entries)
    want = np.frombuffer(g["c2_classes"].encode(), dtype=np.uint8) - ord("0")
    assert np.array_equal(cls, want)
    assert hist.tolist() == g["c2_hist"]
    assert hist[0] == g["c2_zero_count"]["zero_count"]
    assert part[: len(g["c2_partials_head"])].tolist() == g["c2_partials_head"]
    assert gpu.montecarlo_zero(24, 16384, seed=0).zero_count == g["c2_zero_count"]["zero_count"]


def test_c3_structured(gpu):
    g = load_golden("anchors.json")
    from paper_2407_20205_b200 import fixtures

    entries, fam, exp = fixtures.structured_batch(32, 0, 4096)
    cls, _, hist = gpu.perm_mod3_batch(entries)
    known = exp >= 0
    assert np.array_equal(cls[known], exp[known])
    assert hist.sum() == 4096
    if "c3_subset" in g:
        for idx, c in g["c3_subset"]:
            assert cls[idx] == c, idx


def test_c4_c5_windows_and_full(gpu, oracle):
    g = load_golden("anchors.json")
    for key in ("c4_window", "c5_window", "c5_window36"):
        if key not in g:
            continue
        w = g[key]
        m = gpu.MatrixF3(centred(dec(w["a"], w["n"])))
        assert gpu.perm_chunk(m, w["lo"], w["hi"]).partial_sum == w["partial"], key
    if "c4_full" in g:
        w = g["c4_full"]
        m = gpu.MatrixF3(centred(dec(w["a"], 36)))
        assert gpu.perm_chunk(m, 1, 1 << 36).partial_sum == w["partial"]
        assert gpu.perm_mod3_fast(m) % 3 == w["class"]
        # split invariance at full size (the multi-GPU partition rule)
        parts = [gpu.perm_chunk(m, lo, hi).partial_sum for lo, hi in gpu.split_steps(36, 8)]
        assert sum(parts) == w["partial"]


def test_batch_async_device_pointers(gpu):
    import torch

    from paper_2407_20205_b200 import _kernels, fixtures

    for n, B, min_launches in ((14, 257, 1), (21, 65, 3)):  # thread-per-matrix path / pack+walk+finalize
        e = fixtures.uniform_batch(n, 3, 0, B)
        cls_h, part_h, hist_h = gpu.perm_mod3_batch(e)
        d_e = torch.from_numpy(e).cuda()
        d_cls = torch.empty(B, dtype=torch.int8, device="cuda")
        d_pm = torch.empty((B, 2), dtype=torch.int64, device="cuda")
        d_hist = torch.zeros(3, dtype=torch.int64, device="cuda")
        st = torch.cuda.current_stream()
        nl = _kernels.perm_batch_async(d_e.data_ptr(), B, n, d_cls.data_ptr(), d_pm.data_ptr(), d_hist.data_ptr(),
                                       st.cuda_stream)
        torch.cuda.synchronize()
        assert nl >= min_launches
        assert np.array_equal(d_cls.cpu().numpy(), cls_h)
        pm = d_pm.cpu().numpy()
        assert np.array_equal(pm[:, 0] - pm[:, 1], part_h)
        assert d_hist.cpu().tolist() == hist_h.tolist()


def test_abi_rejects_bad_arguments(gpu):
    from paper_2407_20205_b200 import _kernels

    z = np.zeros(4, dtype=np.uint64)
    with pytest.raises(ValueError):
        _kernels.chunk_counts(z, z, 4, 3, 2)
    with pytest.raises(ValueError):
        _kernels.chunk_counts(z, z, 4, 0, 17)
    bad = z.copy()
    bad[0] = 1 << 5
    with pytest.raises(ValueError):
        _kernels.chunk_counts(bad, z, 4, 0, 16)
    with pytest.raises(ValueError):
        _kernels.perm_batch(np.zeros((1, 65, 65), dtype=np.uint8))


def test_integration_binding_from_markdown(gpu):
    """The reference-side ctypes binding shown in INTEGRATION.md works as written."""
    import os
    import re

    from conftest import REPO
    from paper_2407_20205_b200 import _kernels

    md = open(os.path.join(REPO, "INTEGRATION.md")).read()
    code = re.search(r"```python\n(# tritperm/_kernels_b200.py.*?)```", md, flags=re.S).group(1)
    os.environ["TRITPERM_B200_LIB"] = _kernels.LIB_PATH
    ns = {}
    exec(compile(code, "_kernels_b200.py", "exec"), ns)
    for case in load_golden("chunks.json")["cases"][:40]:
        n = case["n"]
        m = gpu.MatrixF3(centred(dec(case["a"], n)))
        mags, sgns = m.planes()
        for lo, hi, s in case["ranges"]:
            if lo >= 1:
                assert ns["chunk_sum"](mags, sgns, n, lo, hi) == s
                assert ns["chunk_sum_devices"](mags, sgns, n, lo, hi, [0]) == s
                assert ns["chunk_sum_devices"](mags, sgns, n, lo, hi, [0], nccl=False) == s
    for case in load_golden("n64.json")["cases"]:  # n = 63, 64 through the same binding
        n = case["n"]
        mags, sgns = gpu.MatrixF3(centred(dec(case["a"], n))).planes()
        for lo, hi, s in case["ranges"]:
            assert ns["chunk_sum"](mags, sgns, n, lo, hi) == s
    for case in load_golden("anchors.json")["montecarlo"][:5]:
        assert ns["mc_zero_count"](case["n"], 0, case["trials"], case["seed"]) == case["zero_count"]
    for case in load_golden("rng.json")["samples"][:8]:
        n = case["n"]
        got = ns["mc_sample_entries"](n, case["trial"], case["seed"]).reshape(n, n)
        assert np.array_equal(np.mod(got.astype(int), 3), dec(case["entries"], n))


def test_distributed_path_single_rank_nccl(gpu, oracle):
    """parallel.py on the device with a real NCCL process group (world size 1:
    the only size a 1-GPU box allows); the 2-rank partition is covered by
    tests/test_parallel_gloo.py."""
    import os
    import socket

    import torch
    import torch.distributed as dist

    from paper_2407_20205_b200 import parallel

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        case = load_golden("anchors.json")["c1"][1]
        a = dec(case["a"], 20)
        m = gpu.MatrixF3(centred(a))
        p, q = parallel.distributed_counts(m)
        assert p - q == case["partial"]
        assert parallel.perm_mod3_distributed(m) % 3 == case["class"]
        h = parallel.distributed_hist([3, 4, 5])
        assert h.tolist() == [3, 4, 5]
    finally:
        dist.destroy_process_group()


def test_pi_matrices_and_pi50_windows(gpu):
    g = load_golden("pi.json")
    for rec in g["pi_matrix"]:
        if "perm" in rec:
            m = gpu.pi_matrix(rec["n"], skip_integer_part=rec["skip_integer_part"])
            assert gpu.perm_mod3_fast(m) == rec["perm"]
            assert gpu.perm_chunk(m, 1, 1 << rec["n"]).partial_sum == rec["partial"]
    for w in g["windows"]:
        m = gpu.pi_matrix(50, skip_integer_part=w["skip_integer_part"])
        assert gpu.perm_chunk(m, w["lo"], w["hi"]).partial_sum == w["partial"]


def test_exact_census_matches_reference_and_paper(gpu):
    """z(1..4) and the +-1 split from the reference's exact_zero_count; z(5)
    from the paper's Table 3 (the reference refuses n = 5)."""
    for rec in load_golden("census.json")["census"]:
        r = gpu.exact_zero_count(rec["n"])
        assert r.z == rec["z"] and r.total == rec["total"], rec
        assert r.z + r.plus_ones + r.minus_ones == r.total
        assert r.plus_ones == r.minus_ones
        if "plus" in rec:
            assert (r.plus_ones, r.minus_ones) == (rec["plus"], rec["minus"])


def _ones_partial(n):
    """Raw Gray partial sum of the all-ones n x n matrix in closed form:
    v_S = |S| (1,...,1), so the term is 0, 1 or (-1)^n for |S| = 0, 1, 2 mod 3."""
    from math import comb

    s = 0
    for k in range(n + 1):
        if k % 3 == 1:
            s += comb(n, k) * (-1) ** k
        elif k % 3 == 2:
            s += comb(n, k) * (-1) ** k * (-1) ** n
    return s


def test_event_dense_matrices_exact(gpu):
    """All-ones matrices: 2/3 of all subsets are full-magnitude events, which
    drives the lane walk's exact mode (n <= 32) and the wide walk's dense mode
    (n > 32) through every superblock; raw partials must stay exact."""
    for n in (14, 20, 24, 31, 32, 33, 34, 36):
        m = gpu.MatrixF3([[1] * n for _ in range(n)])
        assert gpu.perm_chunk(m, 1, 1 << n).partial_sum == _ones_partial(n), n
        assert gpu.perm_mod3_fast(m) == (0 if n >= 3 else 1)
    # dense and sparse matrices mixed in one batch
    from paper_2407_20205_b200 import fixtures

    e = np.concatenate([np.ones((3, 26, 26), np.uint8), fixtures.uniform_batch(26, 9, 0, 3)])
    cls, part, _ = gpu.perm_mod3_batch(e)
    assert part[0] == _ones_partial(26) and cls[0] == 0
    from oracle import oracle as o

    for b in range(3, 6):
        mags, sgns = o.planes_from_classes(e[b])
        assert part[b] == o.chunk_sum(mags, sgns, 26, 1, 1 << 26)


@pytest.mark.parametrize("variant", range(10))
def test_every_fast_walk_variant(gpu, oracle, variant, monkeypatch):
    """Each fast-walk kernel (lane V5/V8, wide, pair narrow/wide V3/V4),
    forced through TRITPERM_FAST_VARIANT, on ranges with heads/tails, a full
    traversal and an event-dense matrix.  A variant that does not fit an n
    falls back to the default, which is also fine."""
    monkeypatch.setenv("TRITPERM_FAST_VARIANT", str(variant))
    r = random.Random(1000 + variant)
    for n in (18, 23, 27, 32, 35, 41, 52):
        a = _rand_matrix(r, n)
        mags, sgns = oracle.planes_from_classes(a)
        m = gpu.MatrixF3(centred(a))
        span = min(1 << 21, 1 << (n - 2))
        lo = r.randrange(1, (1 << n) - 2 * span)
        hi = lo + span + r.randrange(0, 999)
        assert gpu.perm_chunk(m, lo, hi).partial_sum == oracle.chunk_sum(mags, sgns, n, lo, hi), (variant, n)
    a = _rand_matrix(r, 22)
    mags, sgns = oracle.planes_from_classes(a)
    assert gpu.perm_chunk(gpu.MatrixF3(centred(a)), 1, 1 << 22).partial_sum == oracle.chunk_sum(mags, sgns, 22, 1, 1 << 22)
    for n in (24, 34):
        m = gpu.MatrixF3([[1] * n for _ in range(n)])
        assert gpu.perm_chunk(m, 1, 1 << n).partial_sum == _ones_partial(n), (variant, n)


def test_work_queue_resets_between_launches(gpu, oracle):
    """The fast walk's work queue resets itself (last warp out): repeated
    launches on the same stream, a static-assignment plan (few items) and
    CUDA-graph replays all return the same counts."""
    import torch

    from paper_2407_20205_b200 import _kernels, fixtures

    st = torch.cuda.current_stream()
    for n, B in ((20, 1), (24, 300)):  # static items / dynamic queue
        e = fixtures.uniform_batch(n, 7, 0, B)
        d_e = torch.from_numpy(e).cuda()
        d_rows = torch.empty((B, _kernels.ROWREC_BYTES), dtype=torch.uint8, device="cuda")
        d_pm = torch.zeros((B, 2), dtype=torch.int64, device="cuda")
        _kernels.pack_async(d_e.data_ptr(), B, n, d_rows.data_ptr(), st.cuda_stream)
        results = []
        for _ in range(4):
            d_pm.zero_()
            _kernels.walk_async(d_rows.data_ptr(), B, n, d_pm.data_ptr(), st.cuda_stream)
            torch.cuda.synchronize()
            results.append(d_pm.cpu().numpy().copy())
        g = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream()
        side.wait_stream(st)
        with torch.cuda.stream(side):
            _kernels.walk_async(d_rows.data_ptr(), B, n, d_pm.data_ptr(), side.cuda_stream)
        st.wait_stream(side)
        torch.cuda.synchronize()
        with torch.cuda.graph(g):
            _kernels.walk_async(d_rows.data_ptr(), B, n, d_pm.data_ptr(), torch.cuda.current_stream().cuda_stream)
        for _ in range(3):
            d_pm.zero_()
            g.replay()
            torch.cuda.synchronize()
            results.append(d_pm.cpu().numpy().copy())
        for r in results[1:]:
            assert np.array_equal(r, results[0]), n
        for b in (0, B - 1):
            mags, sgns = oracle.planes_from_classes(e[b])
            assert int(results[0][b, 0]) - int(results[0][b, 1]) == oracle.chunk_sum(mags, sgns, n, 1, 1 << n)


def test_filter_pass_heavy_matrices(gpu, oracle):
    """The packed walks filter on 16 columns.  Matrices whose last 16 columns
    are all ones pass that filter for 2/3 of all pairs while real events stay
    rare: the per-superblock verify list overflows and every superblock takes
    the exact fallback without entering dense mode.  Ranges and a batch must
    stay exact (narrow n = 24, 30; wide n = 40)."""
    r = random.Random(4242)
    for n in (24, 30, 40):
        a = _rand_matrix(r, n)
        a[:, n - 16:] = 1
        mags, sgns = oracle.planes_from_classes(a)
        m = gpu.MatrixF3(centred(a))
        for lo, span in ((1 << 22, 1 << 22), (3 << 21, (1 << 22) + 977), (12345, 1 << 21)):
            assert gpu.perm_chunk(m, lo, lo + span).partial_sum == oracle.chunk_sum(mags, sgns, n, lo, lo + span), n
    e = np.stack([_rand_matrix(r, 22) for _ in range(64)])
    e[:, :, 6:] = 1
    _, part, _ = gpu.perm_mod3_batch(e)
    for b in (0, 17, 63):
        mags, sgns = oracle.planes_from_classes(e[b])
        assert part[b] == oracle.chunk_sum(mags, sgns, 22, 1, 1 << 22)


def test_tensor_core_pair_test_exact(gpu, oracle, monkeypatch):
    """The opt-in tcgen05 path (TRITPERM_TC=1, tp_walk_tc.cu): full traversals
    through the batch ABI, n = 18..36 (one and several k-steps, one and two
    32-bit plane words), uniform, all-ones and sparse matrices; raw partials
    equal the oracle's / the default path's bit for bit, and the path's own
    exact re-check of every tensor hit never fires."""
    from paper_2407_20205_b200 import fixtures

    monkeypatch.setenv("TRITPERM_TC", "1")
    r = random.Random(77)
    for n, B in ((18, 40), (21, 9), (24, 64), (29, 3), (32, 2), (33, 1), (36, 1)):
        e = fixtures.uniform_batch(n, 5, 0, B)
        cls, part, hist = gpu.perm_mod3_batch(e)
        monkeypatch.setenv("TRITPERM_TC", "0")
        cls0, part0, hist0 = gpu.perm_mod3_batch(e)
        monkeypatch.setenv("TRITPERM_TC", "1")
        assert np.array_equal(part, part0) and np.array_equal(cls, cls0), n
        assert hist.tolist() == hist0.tolist(), n
        if n <= 24:
            mags, sgns = oracle.planes_from_classes(e[0])
            assert part[0] == oracle.chunk_sum(mags, sgns, n, 1, 1 << n), n
    for n in (20, 24, 31):
        cls, part, _ = gpu.perm_mod3_batch(np.ones((2, n, n), np.uint8))
        assert part[0] == part[1] == _ones_partial(n), n
    sparse = np.array([[[r.choice((0, 0, 0, 0, 1, 2)) for _ in range(22)] for _ in range(22)] for _ in range(8)],
                      dtype=np.uint8)
    _, part, _ = gpu.perm_mod3_batch(sparse)
    for b in range(8):
        mags, sgns = oracle.planes_from_classes(sparse[b])
        assert part[b] == oracle.chunk_sum(mags, sgns, 22, 1, 1 << 22), b


def test_bucketed_pair_walk_exact(gpu, oracle, monkeypatch):
    """The bucketed pair walk on batches (tp_walk_bucket.cu; TRITPERM_BUCKET=1
    packed filter -- 13-row A side / 2 key columns below n = 28, 17 rows / 3
    key columns from n = 28 -- and 2 = unpacked pair tests) against the packed
    walk (TRITPERM_BUCKET=0) and the oracle: full traversals, uniform, sparse
    and all-ones matrices; raw partials bit for bit (only zero terms are
    skipped)."""
    from paper_2407_20205_b200 import fixtures

    r = np.random.default_rng(31)
    cases = [fixtures.uniform_batch(n, 13, 0, B) for n, B in ((21, 48), (22, 7), (24, 40), (27, 3), (31, 2))]
    for n in (21, 26, 29):
        sp = ((r.random((5, n, n)) < 0.25) * r.integers(1, 3, (5, n, n))).astype(np.uint8)
        cases.append(np.concatenate([sp, np.ones((2, n, n), np.uint8)]))
    for e in cases:
        n = e.shape[1]
        monkeypatch.setenv("TRITPERM_BUCKET", "0")
        cls0, part0, hist0 = gpu.perm_mod3_batch(e)
        for mode in ("1", "2"):
            monkeypatch.setenv("TRITPERM_BUCKET", mode)
            cls, part, hist = gpu.perm_mod3_batch(e)
            assert np.array_equal(part, part0) and np.array_equal(cls, cls0), (n, mode)
            assert hist.tolist() == hist0.tolist(), (n, mode)
        if n <= 21:
            mags, sgns = oracle.planes_from_classes(e[0])
            assert part[0] == oracle.chunk_sum(mags, sgns, n, 1, 1 << n), n


def test_bucketed_walk_ranges_and_wide(gpu, oracle, monkeypatch):
    """The bucketed walk on single matrices: n > 32 (primary-word filter, the
    secondary columns checked per pass) and step ranges whose superblock-
    aligned middle it takes while the generic walk takes the unaligned head
    and tail.  Uniform, sparse and all-ones matrices against the oracle and
    the packed walk (TRITPERM_BUCKET=0); the kernel's tested-pair counter
    proves the bucketed walk served the call."""
    from paper_2407_20205_b200 import _kernels

    r = random.Random(77)
    cases = []
    for n in (28, 33, 36, 41, 50):
        cases.append((_rand_matrix(r, n), r.randrange(1, 1 << (n - 3))))
    for n in (34, 39):
        sp = np.array([[r.choice((1, 2)) if r.random() < 0.3 else 0 for _ in range(n)] for _ in range(n)], np.uint8)
        cases.append((sp, r.randrange(1, 1 << 30)))
    cases.append((np.ones((35, 35), np.uint8), 12345))
    for a, lo in cases:
        n = a.shape[0]
        hi = lo + (1 << 27) + r.randrange(0, 1 << 20)
        mags, sgns = oracle.planes_from_classes(a)
        want = oracle.chunk_sum_mt(mags, sgns, n, lo, hi, 8)
        m = gpu.MatrixF3(centred(a))
        monkeypatch.setenv("TRITPERM_BUCKET", "0")
        assert gpu.perm_chunk(m, lo, hi).partial_sum == want, (n, lo, "packed")
        monkeypatch.setenv("TRITPERM_BUCKET", "1")
        _kernels.walk_tested(0)
        assert gpu.perm_chunk(m, lo, hi).partial_sum == want, (n, lo, "bucket")
        assert _kernels.walk_tested(0) > 0, (n, "bucketed walk not used")
    # aligned full traversal above 32 columns, split at arbitrary edges
    a = _rand_matrix(r, 34)
    mags, sgns = oracle.planes_from_classes(a)
    m = gpu.MatrixF3(centred(a))
    full = gpu.perm_chunk(m, 1, 1 << 34).partial_sum
    monkeypatch.setenv("TRITPERM_BUCKET", "0")
    assert gpu.perm_chunk(m, 1, 1 << 34).partial_sum == full
    monkeypatch.setenv("TRITPERM_BUCKET", "1")
    cut = sorted(r.randrange(1, 1 << 34) for _ in range(3))
    edges = [1] + cut + [1 << 34]
    assert sum(gpu.perm_chunk(m, x, y).partial_sum for x, y in zip(edges, edges[1:])) == full
