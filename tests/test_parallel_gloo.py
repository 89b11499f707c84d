"""CPU, world_size 2 over gloo: the multi-GPU partitioning and its single
all-reduce (paper_2407_20205_b200/parallel.py), with the per-rank device
compute replaced by the oracle.  On a B200 box the same code runs with NCCL
and the CUDA counters (bench.py / perm_mod3_parallel under torchrun)."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import REPO, centred, dec, load_golden


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q, tmpdir):
    import sys

    sys.path.insert(0, REPO)
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle
        from paper_2407_20205_b200 import parallel
        from paper_2407_20205_b200.permanent import MatrixF3

        def counts(m, lo, hi):
            mags, sgns = m.planes()
            return oracle.chunk_counts(mags, sgns, m.n, lo, hi)

        out = {}
        g = load_golden("tower.json")
        vals = []
        for block in g["random"][6:12]:  # n = 7..12
            n = block["n"]
            for s, v, partial in block["mats"][:10]:
                m = MatrixF3(centred(dec(s, n)))
                p, q_ = parallel.distributed_counts(m, counts_fn=counts, device="cpu")
                vals.append((p - q_ == partial, parallel.perm_mod3_distributed(m, counts_fn=counts, device="cpu") == v))
        out["tower"] = vals
        # a 20x20 matrix split over the ranks, and an unaligned sub-range
        a = dec(load_golden("anchors.json")["c1"][0]["a"], 20)
        m = MatrixF3(centred(a))
        out["c1"] = parallel.distributed_counts(m, counts_fn=counts, device="cpu")
        out["c1_sub"] = parallel.distributed_counts(m, 12345, 678901, counts_fn=counts, device="cpu")
        # batch shard + histogram all-reduce
        lo_b, hi_b = parallel.shard_rows(37, rank, world)
        local = np.zeros(3, dtype=np.int64)
        for t in range(lo_b, hi_b):
            local[oracle.perm_centered(oracle.sample_classes(8, 5, t)) % 3] += 1
        out["hist"] = parallel.distributed_hist(local.tolist(), device="cpu").tolist()
        out["rank_range"] = parallel.rank_range(20, rank, world)
        # journalled traversal: every part split over the ranks, rank 0 keeps the journal
        from paper_2407_20205_b200 import checkpoint

        def dcounts(mm, lo, hi):
            return parallel.distributed_counts(mm, lo, hi, counts_fn=counts, device="cpu")

        path = os.path.join(tmpdir, "c1.journal")
        first = checkpoint.resumable_counts(m, path, parts=6, max_parts=2, counts_fn=dcounts)
        dist.barrier()
        out["journal_first"] = (first, len(open(path).read().splitlines()))
        dist.barrier()
        out["journal"] = checkpoint.resumable_counts(m, path, parts=6, counts_fn=dcounts)
        dist.barrier()
        out["journal_lines"] = len(open(path).read().splitlines())
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.fixture(scope="module")
def results(oracle, tmp_path_factory):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    tmpdir = str(tmp_path_factory.mktemp("journal"))
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, tmpdir)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


def test_ranks_agree_and_match_reference_tower(results):
    for r in (0, 1):
        assert all(a and b for a, b in results[r]["tower"])


def test_c1_split_over_ranks_matches_single(results, oracle):
    a = dec(load_golden("anchors.json")["c1"][0]["a"], 20)
    mags, sgns = oracle.planes_from_classes(a)
    for r in (0, 1):
        p, q = results[r]["c1"]
        assert p - q == load_golden("anchors.json")["c1"][0]["partial"]
        assert (p, q) == oracle.chunk_counts(mags, sgns, 20, 1, 1 << 20)
        p, q = results[r]["c1_sub"]
        assert p - q == oracle.chunk_sum(mags, sgns, 20, 12345, 678901)


def test_rank_ranges_partition_the_steps(results):
    (a0, a1), (b0, b1) = results[0]["rank_range"], results[1]["rank_range"]
    assert a0 == 1 and a1 == b0 and b1 == 1 << 20


def test_histogram_allreduce(results, oracle):
    want = np.zeros(3, dtype=np.int64)
    for t in range(37):
        want[oracle.perm_centered(oracle.sample_classes(8, 5, t)) % 3] += 1
    assert results[0]["hist"] == results[1]["hist"] == want.tolist()


def test_journalled_traversal_over_ranks(results, oracle):
    """checkpoint.resumable_counts under world_size 2: parts are split over the
    ranks, only rank 0 writes, and a resumed run finishes the missing parts."""
    a = dec(load_golden("anchors.json")["c1"][0]["a"], 20)
    mags, sgns = oracle.planes_from_classes(a)
    want = oracle.chunk_counts(mags, sgns, 20, 1, 1 << 20)
    for r in (0, 1):
        (p, q, complete), lines = results[r]["journal_first"]
        assert not complete and lines == 3  # header + 2 parts, written once
        assert results[r]["journal"] == (want[0], want[1], True)
        assert results[r]["journal_lines"] == 7
